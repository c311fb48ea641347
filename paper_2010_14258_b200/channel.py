"""Seeded link inputs for the bench and the full-size tests, generated on the GPU (§8(f) NEXT-2).

Product-side helper (independent of oracle/channel.py, which the tests compare the GPU SSFM
kernel against): the paper's single-channel link (§IV-A; Table I P:999-1035 with the
readings G16 of DESIGN.md): 16-QAM at 10.7 GBd, RRC roll-off 0.1 shaped on a periodic frame
(Eq. (11)), simulated at rho_a = 4 samples/symbol through 25 x 80 km of SMF by the GPU split-step
kernel (ldbp_ssfm_link: L_eff Kerr + lossy dispersion steps, EDFA gain + ASE drawn in-kernel by
Philox keyed by global block), brick-wall low-pass and decimation to rho_d = 2.  The
training target is the transmitted waveform generated directly at rho_d = 2.

Generation cost is bounded the way SURVEY.md §8(d) prescribes: a pool of U unique simulated
blocks (U / 4 per launch power of the training set P = {-2, -1, 0, 1} dBm), and
global block b uses pool entry (power of b, b mod U/4) circularly shifted by k_b and rotated by
e^{j phi_b} (ldbp_inputs.augment_params) — exact by the shift / phase equivariance of the channel
and of LDBP (pin P10), applied identically to the received block and its target.  Every draw is
keyed by the global block index, so a batch sharded over G ranks is the same batch for any G.
"""
from __future__ import annotations

import math

import numpy as np
import torch

import ldbp_inputs as li

from . import api, init

BAUD_HZ = 10.7e9
RHO_A, RHO_D = 4, 2
SPAN_KM, ALPHA_DB, BETA2_PS2, GAMMA = 80.0, 0.2, -21.7, 1.3
NF_DB, NU_HZ, ROLLOFF = 5.0, 1.946e14, 0.1
H_PLANCK = 6.62607015e-34


def rrc_response(n: int, sps: int, rolloff: float = ROLLOFF, device="cuda") -> torch.Tensor:
    """Root-raised-cosine response on the n-point DFT grid (frequency in cycles/symbol)."""
    f = torch.fft.fftfreq(n, device=device, dtype=torch.float64).abs() * sps
    lo, hi = (1.0 - rolloff) / 2.0, (1.0 + rolloff) / 2.0
    rc = torch.where(f <= lo, torch.ones_like(f),
                     torch.where(f <= hi, 0.5 * (1.0 + torch.cos(math.pi / rolloff * (f - lo))), torch.zeros_like(f)))
    return rc.sqrt()


def modulate(symbols: torch.Tensor, sps: int, power_w: torch.Tensor) -> torch.Tensor:
    """sqrt(P) sum_k s_k p(t - k T) on a periodic frame (Eq. (11)): upsample, RRC in frequency."""
    B, K = symbols.shape
    n = K * sps
    z = torch.zeros((B, n), dtype=torch.complex128, device=symbols.device)
    z[:, ::sps] = symbols.to(torch.complex128)
    x = torch.fft.ifft(torch.fft.fft(z, dim=-1) * rrc_response(n, sps, device=symbols.device), dim=-1)
    return (x * (power_w.to(torch.float64).sqrt() * sps)[:, None]).to(torch.complex64)


def link_constants():
    a = ALPHA_DB * math.log(10.0) / 10.0  # nepers / km
    fs = RHO_A * BAUD_HZ
    n_sp = 0.5 * 10.0 ** (NF_DB / 10.0) * math.exp(a * SPAN_KM) / (math.exp(a * SPAN_KM) - 1.0)
    psd = (math.exp(a * SPAN_KM) - 1.0) * H_PLANCK * NU_HZ * n_sp  # = NF h nu e^{aL} / 2
    return dict(alpha_np=a, beta2=BETA2_PS2 * 1e-24, gamma=GAMMA, fs_hz=fs, span_km=SPAN_KM,
                ase_sigma=math.sqrt(psd * fs))


def simulate_pool(cfg_index: int, U: int, nsym: int, spans: int = 25, stps: int = 50, power_set=(-2, -1, 0, 1),
                  device="cuda"):
    """U unique received blocks [U][RHO_D nsym] and their targets, U / len(power_set) per power."""
    per = U // len(power_set)
    syms, pw = [], []
    for q, p in enumerate(power_set):
        for j in range(per):
            syms.append(li.qam16(li.rng(cfg_index, 1_000_000 + q * per + j, "symbols"), nsym))
            pw.append(float(li.dbm_to_w(p)))
    s = torch.from_numpy(np.stack(syms)).to(device)
    pw_t = torch.tensor(pw, dtype=torch.float64, device=device)
    x = modulate(s, RHO_A, pw_t)
    c = link_constants()
    deltas = init.span_steps(SPAN_KM, stps, ALPHA_DB)
    ws = api.Workspace()
    r = torch.empty((U, RHO_D * nsym), dtype=torch.complex64, device=device)
    chunk = 128
    for a in range(0, U, chunk):
        e = min(U, a + chunk)
        r[a:e] = api.ldbp_ssfm_link(x[a:e].contiguous(), deltas, spans=spans, ase_seed=201014258 + cfg_index,
                                    block0=a, decim=RHO_A // RHO_D, cutoff=0.5 / (RHO_A // RHO_D), ws=ws, **c)
    tgt = modulate(s, RHO_D, pw_t)
    return r, tgt


def link_blocks(cfg_index: int, blocks, n: int, pool=None, U: int = 256, device="cuda"):
    """Received blocks x and targets [len(blocks)][n] for global block indices `blocks` (n = 2 nsym)."""
    blocks = list(blocks)
    if pool is None:
        pool = simulate_pool(cfg_index, U, n // RHO_D, device=device)
    r, tgt = pool
    U = r.shape[0]
    per = U // 4
    q = np.searchsorted(np.array([-2.0, -1.0, 0.0, 1.0]), li.pick_powers_dbm(cfg_index, blocks, (-2.0, -1.0, 0.0, 1.0)))
    idx = torch.from_numpy(q * per + np.array(blocks) % per).to(device)
    ks, phis = li.augment_params(cfg_index, blocks, n)
    k = torch.from_numpy(ks).to(device)
    ph = torch.polar(torch.ones(len(blocks), dtype=torch.float64, device=device),
                     torch.from_numpy(phis).to(device)).to(torch.complex64)
    cols = (torch.arange(n, device=device)[None, :] - k[:, None]) % n  # roll by k_b: out[t] = in[t - k]
    x = torch.empty((len(blocks), n), dtype=torch.complex64, device=device)
    t = torch.empty_like(x)
    for a in range(0, len(blocks), 1024):
        e = min(len(blocks), a + 1024)
        x[a:e] = torch.gather(r[idx[a:e]], 1, cols[a:e]) * ph[a:e, None]
        t[a:e] = torch.gather(tgt[idx[a:e]], 1, cols[a:e]) * ph[a:e, None]
    return x, t


def qam16_table(device="cuda") -> torch.Tensor:
    """complex64 [16] constellation of ldbp_inputs.qam16_codes (code 4 i + q)."""
    return torch.from_numpy(li.QAM16_TABLE.astype(np.complex64)).to(device)


def link_codes(cfg_index: int, blocks, n: int, U: int = 256, device="cuda"):
    """What a training step needs to rebuild link_blocks' targets on the device
    (api.ldbp_tx_waveform): uint8 symbol codes [len(blocks)][n / RHO_D] of each block's pool entry,
    its launch power (W, float32), circular shift (int32) and rotation (rad, float32)."""
    blocks = list(blocks)
    nsym = n // RHO_D
    per = U // 4
    pset = (-2.0, -1.0, 0.0, 1.0)
    q = np.searchsorted(np.array(pset), li.pick_powers_dbm(cfg_index, blocks, pset))
    pool = q * per + np.array(blocks) % per
    codes = np.stack([li.qam16_codes(li.rng(cfg_index, 1_000_000 + int(p), "symbols"), nsym) for p in pool])
    pw = np.array([float(li.dbm_to_w(pset[int(qq)])) for qq in q], dtype=np.float32)
    ks, phis = li.augment_params(cfg_index, blocks, n)
    return (torch.from_numpy(codes).to(device), torch.from_numpy(pw).to(device),
            torch.from_numpy(np.asarray(ks, dtype=np.int32)).to(device),
            torch.from_numpy(np.asarray(phis, dtype=np.float32)).to(device))
