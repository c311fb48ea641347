"""C1 training-step latency with the whole step (loss_grad + Adam) in one CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print("C1 graph us/step %.2f" % bench.graph_latency(bench.CONFIGS["C1"]))
