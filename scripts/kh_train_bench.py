"""Training-step kernel times at a C3-like shape with another filter length:
    python scripts/kh_train_bench.py T [T ...]   (LDBP_LIB selects the library)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402
from paper_2010_14258_b200 import _lib  # noqa: E402

for T in [int(t) for t in sys.argv[1:]] or [5, 7]:
    cfg = dict(bench.CONFIGS["C3"], T=T)
    taps, gamma = bench.make_model(cfg)
    x, tgt = bench.make_inputs(cfg, range(cfg["B"]))
    st = P.TrainState.create(taps, gamma)
    ws = P.Workspace()
    for _ in range(3):
        P.ldbp_loss_grad(x, tgt, st.taps, st.gamma, ws=ws)
    torch.cuda.synchronize()
    per = {}
    reps = 10
    with P.api.trace() as tr:
        for _ in range(reps):
            P.ldbp_loss_grad(x, tgt, st.taps, st.gamma, ws=ws)
        torch.cuda.synchronize()
    for kind, steps, samples, ms in tr.records:
        per[kind] = per.get(kind, 0.0) + ms
    print(f"T={T}: forward {per.get(_lib.K_FORWARD, 0) / reps:.3f} ms, reverse {per.get(_lib.K_REVERSE, 0) / reps:.3f} ms")
