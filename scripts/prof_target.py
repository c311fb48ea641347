"""Run one warm and one measured launch set of a bench configuration (profiling target).

    python scripts/prof_target.py C2|C3|C4|C5 [reps]

Env: PROF_B=<blocks> overrides the batch, PROF_FWD=1 runs the forward only.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = dict(bench.CONFIGS[name])
if os.environ.get("PROF_B"):
    cfg["B"] = int(os.environ["PROF_B"])
if os.environ.get("PROF_FWD"):
    cfg["mode"] = "fwd"
taps, gamma = bench.make_model(cfg)
x, tgt = bench.make_inputs(cfg, range(cfg["B"]))
st = P.TrainState.create(taps, gamma)
for _ in range(reps):
    if cfg["mode"] == "train":
        buf = P.ldbp_train_step(st, x, tgt)
    else:
        y = P.ldbp_forward(x, st.taps, st.gamma)
torch.cuda.synchronize()
print("ok", name)
