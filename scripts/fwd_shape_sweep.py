"""Forward-kernel fraction of the FP32 peak vs (B, M) at n = 2^14, T = 5 (C2's filter):
separates per-launch overhead (load, prologue, store; fixed per launch) from the step loop.

    python scripts/fwd_shape_sweep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ws = P.Workspace()
for B, M in [(256, 25), (256, 50), (256, 100), (512, 25), (1024, 25), (128, 25)]:
    cfg = dict(bench.CONFIGS["C2"], B=B)
    x, _ = bench.make_inputs(cfg, range(cfg["B"]))
    taps, gamma = bench.make_model(cfg)
    reps = -(-M // taps.shape[0])
    taps = np.concatenate([taps] * reps)[:M]
    gamma = np.concatenate([gamma] * reps)[:M]
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
    kh = (taps.shape[1] - 1) // 2
    ss = B * cfg["n"] * M
    frac = ss * (6 * kh + 12) / (ms * 1e-3) / (148 * 128 * 1.965e9)
    print(f"B={B} M={M}: {ms * 1e3:.1f} us  {ss / ms / 1e6:.1f} Gss/s  frac {frac:.3f}")
    del x
