"""C1 training-step latency, the whole step (ldbp_train_step) in a CUDA graph: 20 steps per graph
(device time) and, for comparison, one step per graph (bounded by the host's replay rate)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for nm in ("C1", "C2"):
    c = bench.CONFIGS[nm]
    print("%s graph us/step: %.2f (20 steps/graph)  %.2f (1 step/graph)"
          % (nm, bench.graph_latency(c), bench.graph_latency(c, reps=50, inner=1)))
