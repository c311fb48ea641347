"""C1 training steps (the fused tiny kernel) for an ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

c = bench.CONFIGS["C1"]
taps, gamma = bench.make_model(c)
x, tgt = bench.make_inputs(c, range(c["B"]))
st = P.TrainState.create(taps, gamma)
for _ in range(6):
    P.ldbp_train_step(st, x, tgt)
torch.cuda.synchronize()
print("ok")
