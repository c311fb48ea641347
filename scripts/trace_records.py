"""Print the traced launches (kind, steps, samples, ms) of one C3 loss_grad + Adam step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = bench.CONFIGS[name]
taps, gamma = bench.make_model(cfg)
x, tgt = bench.make_inputs(cfg, 0)
st = P.TrainState.create(taps, gamma)
buf = P.ldbp_loss_grad(x, tgt, st.taps, st.gamma)
torch.cuda.synchronize()
with P.api.trace() as tr:
    buf = P.ldbp_loss_grad(x, tgt, st.taps, st.gamma)
    P.ldbp_adam_update(st, buf, cfg["B"] * cfg["n"])
    torch.cuda.synchronize()
for r in tr.records:
    print(r)
