"""§8(f) NEXT-4 cost: learned ESSM (kappa = 20) forward and loss+gradient at a C3-like shape
(512 blocks x 2^14, M = 25, T = 9), one launch per step, vs the fused LDBP kernels.

    python scripts/essm_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

cfg = dict(bench.CONFIGS["C3"])
B, n, M, T, kap = cfg["B"], cfg["n"], 25, 9, 20
cfg.update(sps=1)
taps, gamma = bench.make_model(cfg)
taps, gamma = taps[:M], gamma[:M]
x, tgt = bench.make_inputs(cfg, range(cfg["B"]))
eta = np.ones((M, 2 * kap + 1)) / (2 * kap + 1)
ht = torch.from_numpy(taps.astype(np.complex64)).cuda()
gt = torch.from_numpy(gamma.astype(np.float32)).cuda()
et = torch.from_numpy(eta.astype(np.float32)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ws = P.Workspace()


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.fill_(1.0)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / reps


ss = B * n * M
for name, fn in (("ESSM forward", lambda: P.ldbp_essm_forward(x, ht, gt, et, ws=ws)),
                 ("ESSM loss+grad", lambda: P.ldbp_essm_loss_grad(x, tgt, ht, gt, et, ws=ws)),
                 ("LDBP forward (same M, T)", lambda: P.ldbp_forward(x, ht, gt, ws=ws)),
                 ("LDBP loss+grad (same M, T)", lambda: P.ldbp_loss_grad(x, tgt, ht, gt, ws=ws))):
    t = timed(fn)
    print(f"{name:28s} {t:8.3f} ms  {ss / t / 1e6:8.1f} Gsample-steps/s")
