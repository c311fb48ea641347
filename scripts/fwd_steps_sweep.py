"""C2-shaped inference forward (256 x 2^14, T = 5) at M = 1 .. 50: per-step slope and fixed cost.
    python scripts/fwd_steps_sweep.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ldbp_inputs as li  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

B, n, T = int(os.environ.get("SWEEP_B", 256)), 16384, 5
x = torch.from_numpy(li.bandlimited_blocks(2, range(B), n, 1e-3).astype(np.complex64)).cuda()
ws = P.Workspace()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for M in [int(m) for m in os.environ.get("SWEEP_M", "1,2,5,12,25,50").split(",")]:
    taps = torch.from_numpy(li.random_sym_taps(2, M, T, 0.05).astype(np.complex64)).cuda()
    gam = torch.from_numpy(li.random_gamma(2, M).astype(np.float32)).cuda()
    y = torch.empty_like(x)
    for _ in range(3):
        P.ldbp_forward(x, taps, gam, out=y, ws=ws)
    torch.cuda.synchronize()
    with P.api.trace() as tr:
        for i in range(10):
            flush.fill_(i)
            P.ldbp_forward(x, taps, gam, out=y, ws=ws)
        torch.cuda.synchronize()
    ms = sum(r[3] for r in tr.records) / 10
    print(f"M={M:3d}: {ms * 1e3:8.1f} us  {ms * 1e3 / M:7.2f} us/step  launches/call {len(tr.records) / 10:.0f}")
