"""Profiling target: C2-shaped inference forward (256 x 2^14, T = 5) with M steps (argv[1])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ldbp_inputs as li  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 25
B, n, T = 256, 16384, 5
x = torch.from_numpy(li.bandlimited_blocks(2, range(B), n, 1e-3).astype(np.complex64)).cuda()
taps = torch.from_numpy(li.random_sym_taps(2, M, T, 0.05).astype(np.complex64)).cuda()
gam = torch.from_numpy(li.random_gamma(2, M).astype(np.float32)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    P.ldbp_forward(x, taps, gam, out=y)
torch.cuda.synchronize()
print("ok")
