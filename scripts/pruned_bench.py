"""§8(f) NEXT-3 evidence: C3-shaped training step and forward with a pruned model (per-step
active half-lengths alternating 4/2, i.e. 9/5 taps) vs the unpruned model, same kernels.

    python scripts/pruned_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

cfg = bench.CONFIGS["C3"]
taps, gamma = bench.make_model(cfg)
M, T = taps.shape
kh = (T - 1) // 2
x, tgt = bench.make_inputs(cfg, range(cfg["B"]))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ws = P.Workspace()


def timed(fn, reps=10):
    for _ in range(3):
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


for name, pattern in (("unpruned", [kh] * M), ("pruned 9/5", [kh if i % 2 == 0 else kh - 2 for i in range(M)]),
                      ("pruned 5/3", [2 if i % 2 == 0 else 1 for i in range(M)])):
    mask = np.ones((M, T), np.uint8)
    for i, k in enumerate(pattern):
        for j in range(k + 1, kh + 1):
            mask[i, kh + j] = mask[i, kh - j] = 0
    ht = torch.from_numpy((taps * mask).astype(np.complex64)).cuda()
    gt = torch.from_numpy(gamma.astype(np.float32)).cuda()
    mt = torch.from_numpy(mask).cuda()
    active = int(mask.sum())
    t_f = timed(lambda: P.ldbp_forward(x, ht, gt, ws=ws))
    st = P.TrainState.create(taps * mask, gamma, mask=mask)
    t_g = timed(lambda: P.ldbp_loss_grad_state(st, x, tgt, ws=ws))  # active-window training (NEXT-3)
    ss = cfg["B"] * cfg["n"] * M
    print(f"{name:12s} active taps {active:4d}: forward {t_f:.3f} ms ({ss / t_f / 1e6:.1f} Gss/s), "
          f"loss+grad {t_g:.3f} ms ({ss / t_g / 1e6:.1f} Gss/s)")
