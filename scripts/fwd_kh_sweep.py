"""Forward-kernel throughput vs filter half-length Kh at the C3 shape (512 x 2^14, M = 50),
fraction of the FP32 peak with the algorithmic 6Kh+12 lane-ops per sample-step.

    python scripts/fwd_kh_sweep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

cfg = dict(bench.CONFIGS["C3"])
x, _ = bench.make_inputs(cfg, range(cfg["B"]))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ws = P.Workspace()
for T in (3, 5, 7, 9, 11, 13, 15):
    cfg["T"] = T
    taps, gamma = bench.make_model(cfg)
    ht = torch.from_numpy(taps.astype(np.complex64)).cuda()
    gt = torch.from_numpy(gamma.astype(np.float32)).cuda()
    for _ in range(3):
        P.ldbp_forward(x, ht, gt, ws=ws)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in ev:
        flush.fill_(1.0)
        a.record()
        P.ldbp_forward(x, ht, gt, ws=ws)
        b.record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)
    kh = (T - 1) // 2
    ss = cfg["B"] * cfg["n"] * len(gamma)
    frac = ss * (6 * kh + 12) / (ms * 1e-3) / (148 * 128 * 1.965e9)
    print(f"Kh={kh}: {ms:.3f} ms  {ss / ms / 1e6:.1f} Gss/s  frac {frac:.3f}")
