"""§8(f) NEXT-2 cost: GPU SSFM generator, 512 blocks x 2^14 samples (4096 16-QAM symbols at
rho_a = 4), 25 spans x 8 steps + EDFA/ASE + LPF/decimation to 2 sps, vs the numpy oracle on one block.

    python scripts/ssfm_bench.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ldbp_inputs as li  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402
from oracle import channel, physics, steps  # noqa: E402

B, nsym, rho_a, spans, S = 512, 4096, 4, 25, 8
n = nsym * rho_a
a = physics.alpha_np_per_km(0.2)
prm = dict(alpha_np=a, beta2=physics.ps2_per_km(-21.7), gamma=1.3, fs_hz=rho_a * 10.7e9, span_km=80.0)
sig = float(np.sqrt(physics.ase_psd(5.0, a, 80.0, 1.946e14) * prm["fs_hz"]))
deltas = steps.log_step_sizes(80.0, S, a)
s = np.stack([li.qam16(li.rng(5, b, "symbols"), nsym) for b in range(4)])
x0 = np.stack([channel.modulate(s[b], rho_a, 1e-3) for b in range(4)])
x = torch.from_numpy(np.tile(x0, (B // 4, 1)).astype(np.complex64)).cuda()
noise = (torch.randn(spans, B, n, 2, device="cuda") * np.sqrt(0.5)).view(torch.complex64).squeeze(-1).contiguous()
ws = P.Workspace()


def run():
    u = x.clone()
    return P.ldbp_ssfm_link(u, deltas, spans=spans, ase_sigma=sig, noise=noise, decim=2, cutoff=0.25, ws=ws, **prm)


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
steps_total = spans * S
ffts = 2 * steps_total + 2
gflops = B * ffts * 5 * n * np.log2(n) / (ms * 1e-3) / 1e9
print(f"GPU SSFM: {ms:.2f} ms for {B} blocks x {n} samples x {steps_total} steps "
      f"({B * n * steps_total / ms / 1e6:.1f} Gsample-steps/s, {gflops:.0f} GFLOP/s of FFT work)")
t0 = time.time()
u = x0[:1].astype(np.complex128)
for k in range(spans):
    u = channel.ssfm(u, deltas, a, prm["beta2"], prm["gamma"], prm["fs_hz"])
    u = channel.edfa(u, a, 80.0, sig ** 2 / prm["fs_hz"], prm["fs_hz"], None)
t = time.time() - t0
print(f"oracle (numpy fp64, 1 core): {t * 1e3:.0f} ms per block -> {t * B:.1f} s for the batch "
      f"(GPU speed-up {t * B / (ms * 1e-3):.0f}x)")
