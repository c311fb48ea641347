"""§8(f) NEXT-1 cost at C3 size: receiver-chain loss+gradient alone, and the receiver-chain
training gradient (storing forward + MF/phase/adjoint + reverse) vs the waveform-MSE one.

    python scripts/rx_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import ldbp_inputs as li  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402
from paper_2010_14258_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS["C3"]
B, n = cfg["B"], cfg["n"]
sps, span = 2, 32
taps, gamma = bench.make_model(cfg)
M, T = taps.shape
x, tgt = bench.make_inputs(cfg, range(cfg["B"]))
sym = torch.from_numpy(np.stack([li.qam16(li.rng(3, b, "symbols"), n // sps) for b in range(B)])
                       .astype(np.complex64)).cuda()
pw = torch.full((B,), 1e-3, dtype=torch.float32, device="cuda")
# RRC matched-filter taps (reading G19): periodic RRC impulse response truncated to +-span symbols
L = span * sps
nref = 1 << 18
f = np.abs(np.fft.fftfreq(nref) * sps)
lo, hi = 0.45, 0.55
rc = np.where(f <= lo, 1.0, np.where(f <= hi, 0.5 * (1.0 + np.cos(np.pi / 0.1 * (f - lo))), 0.0))
hh = np.fft.ifft(np.sqrt(rc)).real
h = torch.from_numpy(np.concatenate([hh[-L:], hh[:L + 1]]).astype(np.float32)).cuda()
ht = torch.from_numpy(taps.astype(np.complex64)).cuda()
gt = torch.from_numpy(gamma.astype(np.float32)).cuda()
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


t_rx = timed(lambda: P.ldbp_rx_loss_grad(x, sym, pw, h, sps=sps, ws=ws))
with P.api.trace() as tr:
    P.ldbp_rx_loss_grad(x, sym, pw, h, sps=sps, ws=ws)
    torch.cuda.synchronize()
t_mse = timed(lambda: P.ldbp_loss_grad(x, tgt, ht, gt, ws=ws))
t_rxt = timed(lambda: P.ldbp_rx_train_grad(x, sym, pw, h, ht, gt, sps=sps, ws=ws))
ss = B * n * M
# MF + adjoint: (2L+1) real taps per symbol each way, 2 lane-ops (FFMA2) per tap -> per sample
lane_ops = 2 * (2 * L + 1) * 2 * (n // sps) * B
print(f"rx loss+grad alone: {t_rx:.3f} ms  ({lane_ops / (t_rx * 1e-3) / (148 * 128 * 1.965e9):.3f} of FP32 peak; "
      f"launches {[(k, round(ms, 3)) for k, _, _, ms in tr.records]})")
print(f"waveform-MSE train grad: {t_mse:.3f} ms ({ss / t_mse / 1e6:.1f} Gss/s)")
print(f"receiver-chain train grad: {t_rxt:.3f} ms ({ss / t_rxt / 1e6:.1f} Gss/s)")
t_rxe = timed(lambda: P.ldbp_rx_exact_loss_grad(x, sym, pw, sps=sps))
t_rxet = timed(lambda: P.ldbp_rx_exact_train_grad(x, sym, pw, ht, gt, sps=sps, ws=ws))
# 4 FFTs of n points per block (5 n log2 n flops each): MF forward + inverse, adjoint forward + inverse
fft_flops = 4 * 5 * n * np.log2(n) * B
print(f"exact circulant MF loss+grad alone: {t_rxe:.3f} ms ({fft_flops / (t_rxe * 1e-3) / 1e12:.2f} TFLOP/s of FFT work)")
print(f"receiver-chain train grad, exact MF: {t_rxet:.3f} ms ({ss / t_rxet / 1e6:.1f} Gss/s)")
