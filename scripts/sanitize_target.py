"""Small calls of every hot-path kernel for compute-sanitizer (racecheck / synccheck / memcheck):
store-all schedule (params, storing forward, reverse, two-level reduction), segment schedule,
forward, Adam, the exact receiver and the SSFM cluster kernel.

    compute-sanitizer --tool racecheck python scripts/sanitize_target.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ldbp_inputs as li  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402

B, n, M, T = 6, 4096, 4, 5
x = torch.from_numpy(li.gaussian_blocks(1, range(B), n, 1e-3).astype(np.complex64)).cuda()
t = torch.from_numpy(li.gaussian_blocks(1, range(B), n, 1e-3, purpose="target").astype(np.complex64)).cuda()
st = P.TrainState.create(li.random_sym_taps(1, M, T, 0.05), li.random_gamma(1, M))
y = P.ldbp_forward(x, st.taps, st.gamma)
for mode in ("1", "0", "1r4"):
    os.environ["LDBP_REV4"] = "1" if mode == "1r4" else "0"  # shared-memory-adjoint reverse too
    mode = mode[:1]
    os.environ["LDBP_BWD_MODE"] = mode
    os.environ["LDBP_STORE_ALL_MIN_SAMPLES"] = "0"
    os.environ["LDBP_REV_MAX_STEPS"] = "2"  # two reverse launches (adjoint through HBM)
    buf = P.ldbp_loss_grad(x, t, st.taps, st.gamma)
    P.ldbp_adam_update(st, buf, B * n)
sym = torch.from_numpy(np.stack([li.qam16(li.rng(1, b, "symbols"), n // 2) for b in range(B)]).astype(np.complex64)).cuda()
pw = torch.full((B,), 1e-3, dtype=torch.float32, device="cuda")
P.ldbp_rx_exact_loss_grad(y, sym, pw, sps=2)
u = torch.from_numpy(li.gaussian_blocks(2, range(2), 1 << 15, 1e-3).astype(np.complex64)).cuda()
P.ldbp_ssfm_link(u, [40.0, 40.0], spans=1, span_km=80.0, alpha_np=0.046, beta2=-21.7e-24, gamma=1.3, fs_hz=42.8e9,
                 ase_sigma=1e-4, ase_seed=3)
torch.cuda.synchronize()
print("sanitize target done")
