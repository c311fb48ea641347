"""Seeded synthetic input generators shared by the tests, the oracle's callers and bench.py.

This module holds ONLY random draws and their plumbing (seed streams, symbol alphabets,
circular-Gaussian noise, power picks, random taps).  It contains none of the LDBP method's
arithmetic (no FIR, no Kerr rotation, no split-step, no gradient), so both the CPU oracle
(`oracle/`) and the CUDA path can consume its output without sharing method code.

Seed tree (SURVEY.md §8(d) "Seeds"): each configuration's root is
``SeedSequence([201014258, cfg_index])``; every draw is keyed by
``(global block index, purpose)`` so that the union of the blocks a rank generates is
identical for any number of ranks G.
"""
from __future__ import annotations

import numpy as np

SEED_ROOT = 201014258

# purpose ids for the keyed streams (stable numbering; never reorder)
PURPOSES = {
    "symbols": 1,
    "ase": 2,
    "taps": 3,
    "power": 4,
    "augment": 5,
    "signal": 6,
    "target": 7,
    "gamma": 8,
    "grad": 9,
}


def rng(cfg_index: int, block: int, purpose: str, sub: int = 0) -> np.random.Generator:
    """Independent PCG64 stream keyed by (config, global block index, purpose, sub-key)."""
    ss = np.random.SeedSequence([SEED_ROOT, int(cfg_index), int(block), PURPOSES[purpose], int(sub)])
    return np.random.Generator(np.random.PCG64(ss))


def cn(g: np.random.Generator, shape) -> np.ndarray:
    """Circularly-symmetric complex Gaussian CN(0, 1) draws (E|z|^2 = 1), complex128."""
    re = g.standard_normal(shape)
    im = g.standard_normal(shape)
    return (re + 1j * im) * np.sqrt(0.5)


QAM16_LEVELS = np.array([-3.0, -1.0, 1.0, 3.0]) / np.sqrt(10.0)


def qam16(g: np.random.Generator, count: int) -> np.ndarray:
    """Uniform iid 16-QAM symbols, per-dimension levels {+-1, +-3}/sqrt(10) (unit mean power)."""
    i = g.integers(0, 4, size=count)
    q = g.integers(0, 4, size=count)
    return QAM16_LEVELS[i] + 1j * QAM16_LEVELS[q]


# code 4 i + q  <->  QAM16_LEVELS[i] + j QAM16_LEVELS[q]
QAM16_TABLE = (QAM16_LEVELS[:, None] + 1j * QAM16_LEVELS[None, :]).reshape(-1)


def qam16_codes(g: np.random.Generator, count: int) -> np.ndarray:
    """The same draws as qam16(g, count) as uint8 codes into QAM16_TABLE."""
    i = g.integers(0, 4, size=count)
    q = g.integers(0, 4, size=count)
    return (4 * i + q).astype(np.uint8)


def dbm_to_w(p_dbm):
    return 10.0 ** ((np.asarray(p_dbm, dtype=np.float64) - 30.0) / 10.0)


def pick_powers_dbm(cfg_index: int, blocks, power_set_dbm) -> np.ndarray:
    """Per-block launch power drawn uniformly from the discrete set P (paper P:839-843)."""
    ps = np.asarray(power_set_dbm, dtype=np.float64)
    return np.array([ps[rng(cfg_index, b, "power").integers(0, len(ps))] for b in blocks])


def gaussian_blocks(cfg_index: int, blocks, n: int, power_w, purpose: str = "signal") -> np.ndarray:
    """complex128 [len(blocks)][n] circular-Gaussian blocks with mean power power_w[b] (W).

    After 2000 km of chromatic dispersion the received samples are close to circular complex
    Gaussian with the launch power (SURVEY.md §8(d) "Value distribution"); this is the bench's
    stand-in for SSFM output at sizes the CPU channel simulator cannot produce in time.
    """
    blocks = list(blocks)
    pw = np.broadcast_to(np.asarray(power_w, dtype=np.float64), (len(blocks),))
    out = np.empty((len(blocks), n), dtype=np.complex128)
    for i, b in enumerate(blocks):
        out[i] = cn(rng(cfg_index, b, purpose), n) * np.sqrt(pw[i])
    return out


def random_sym_taps(cfg_index: int, steps: int, taps: int, scale: float = 0.1) -> np.ndarray:
    """Seeded symmetric taps h = delta_0 + scale*CN(0,1) on the half taps.

    Returned as complex128 [steps][taps], tap j in [-Kh, Kh] stored at index j+Kh.
    """
    kh = (taps - 1) // 2
    g = rng(cfg_index, 0, "taps")
    half = cn(g, (steps, kh + 1)) * scale
    half[:, 0] += 1.0
    full = np.empty((steps, taps), dtype=np.complex128)
    for j in range(kh + 1):
        full[:, kh + j] = half[:, j]
        full[:, kh - j] = half[:, j]
    return full


def random_general_taps(cfg_index: int, steps: int, taps: int, scale: float = 0.1, sub: int = 0) -> np.ndarray:
    """Seeded non-symmetric taps delta_0 + scale*CN(0,1) on all T taps, complex128 [steps][taps]."""
    kh = (taps - 1) // 2
    g = rng(cfg_index, 0, "taps", sub=1000 + sub)
    full = cn(g, (steps, taps)) * scale
    full[:, kh] += 1.0
    return full


def random_gamma(cfg_index: int, steps: int, lo: float = -30.0, hi: float = -5.0, sub: int = 0) -> np.ndarray:
    """Seeded per-step signed nonlinearity scalars gamma' (1/W), uniform in [lo, hi]."""
    g = rng(cfg_index, 0, "gamma", sub=sub)
    return g.uniform(lo, hi, size=steps)


def augment_params(cfg_index: int, blocks, n: int):
    """Per-block (circular shift k_b, phase phi_b) for the equivariant pool augmentation (§8(d))."""
    ks, phis = [], []
    for b in blocks:
        g = rng(cfg_index, b, "augment")
        ks.append(int(g.integers(0, n)))
        phis.append(float(g.uniform(-np.pi, np.pi)))
    return np.array(ks, dtype=np.int64), np.array(phis)


def to_complex64(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex64)


# ---------------------------------------------------------------------------------------
# Band-limited circular Gaussian waveforms (bench / full-size tests)
# ---------------------------------------------------------------------------------------
# A 16-QAM RRC signal after ~2000 km of chromatic dispersion is, by the CLT over the ~69-symbol
# CD memory (Eq. 15), close to a circular Gaussian process whose spectrum fills the
# RRC band |f| <= (1 + rolloff) R_s / 2.  At rho_d = 2 samples/symbol that is the
# fraction OCCUPIED = (1 + 0.1) / 2 of the sampling band.  These generators draw such blocks
# directly (no channel arithmetic): white CN(0,1) -> keep the occupied DFT bins -> unit power
# -> scale by sqrt(P_b).
OCCUPIED = (1.0 + 0.1) / 2.0


def bandlimited_mask(n: int, occupied: float = OCCUPIED) -> np.ndarray:
    f = np.fft.fftfreq(n)
    return (np.abs(f) <= occupied / 2.0).astype(np.float64)


def bandlimited_blocks(cfg_index: int, blocks, n: int, power_w, occupied: float = OCCUPIED,
                       purpose: str = "signal") -> np.ndarray:
    """numpy complex128 [len(blocks)][n] band-limited circular Gaussian blocks, mean power power_w[b]."""
    w = gaussian_blocks(cfg_index, blocks, n, 1.0, purpose)
    m = bandlimited_mask(n, occupied)
    out = np.fft.ifft(np.fft.fft(w, axis=-1) * m, axis=-1) * np.sqrt(n / m.sum())
    pw = np.broadcast_to(np.asarray(power_w, dtype=np.float64), (len(list(blocks)),))
    return out * np.sqrt(pw)[:, None]


def bandlimited_blocks_torch(seed: int, B: int, n: int, power_w, device="cuda", occupied: float = OCCUPIED,
                             chunk: int = 512):
    """Same recipe drawn on the device with a seeded torch generator (complex64 [B][n]).

    ``power_w``: scalar or length-B sequence of per-block powers (W).  Generated in chunks of
    blocks so the FFT scratch stays small at the 2^28-sample configurations."""
    import torch

    g = torch.Generator(device=device).manual_seed(int(seed))
    out = torch.empty((B, n), dtype=torch.complex64, device=device)
    f = torch.fft.fftfreq(n, device=device)
    mask = (f.abs() <= occupied / 2.0).to(torch.complex64)
    norm = float(np.sqrt(n / float(mask.real.sum().item())))
    pw = torch.as_tensor(np.broadcast_to(np.asarray(power_w, dtype=np.float64), (B,)).copy(), device=device)
    amp = (pw.sqrt() * norm).to(torch.float32)
    for s in range(0, B, chunk):
        e = min(B, s + chunk)
        w = torch.randn((e - s, n), dtype=torch.complex64, device=device, generator=g)
        out[s:e] = torch.fft.ifft(torch.fft.fft(w, dim=-1) * mask, dim=-1) * amp[s:e, None]
    return out


def bandlimited_blocks_keyed_torch(cfg_index: int, blocks, n: int, power_w, device="cuda",
                                   occupied: float = OCCUPIED, chunk: int = 256, purpose: str = "signal"):
    """Band-limited circular Gaussian blocks (recipe above) drawn on the device, one seeded torch
    generator per GLOBAL block index: block b's samples depend only on (cfg_index, b, purpose),
    so the union over ranks of a sharded batch is the same for any number of ranks G
    (SURVEY.md §8(e)).  complex64 [len(blocks)][n]; ``power_w`` scalar or per listed block."""
    import torch

    blocks = list(blocks)
    B = len(blocks)
    out = torch.empty((B, n), dtype=torch.complex64, device=device)
    f = torch.fft.fftfreq(n, device=device)
    mask = (f.abs() <= occupied / 2.0).to(torch.complex64)
    norm = float(np.sqrt(n / float(mask.real.sum().item())))
    pw = torch.as_tensor(np.broadcast_to(np.asarray(power_w, dtype=np.float64), (B,)).copy(), device=device)
    amp = (pw.sqrt() * norm).to(torch.float32)
    g = torch.Generator(device=device)
    w = torch.empty((min(chunk, max(B, 1)), n), dtype=torch.complex64, device=device)
    for s in range(0, B, chunk):
        e = min(B, s + chunk)
        for i in range(s, e):
            key = np.random.SeedSequence([SEED_ROOT, int(cfg_index), int(blocks[i]), PURPOSES[purpose]])
            g.manual_seed(int(key.generate_state(1, dtype=np.uint64)[0] >> 1))
            torch.randn((n,), dtype=torch.complex64, device=device, generator=g, out=w[i - s])
        out[s:e] = torch.fft.ifft(torch.fft.fft(w[: e - s], dim=-1) * mask, dim=-1) * amp[s:e, None]
    return out


# ---------------------------------------------------------------------------------------
# Counter-based ASE draws (shared generator: the GPU channel kernel implements the same Philox)
# ---------------------------------------------------------------------------------------
# Philox4x32-10 (Salmon et al., SC'11): counter (c0, c1, c2, c3), key (k0, k1); per round
#   (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2,  c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0),
#   key <- key + (W0, W1).
# The ASE draw of sample i of span `span` of global block `block` (SURVEY.md §8(d) seed tree:
# keyed by global block index, so the union is independent of the number of ranks) is
#   x = philox((i >> 1, span, block & 0xffffffff, block >> 32), (seed & 0xffffffff, seed >> 32)),
#   (u1, u2) = ((x0 + 0.5) 2^-32, (x1 + 0.5) 2^-32) for even i, (x2, x3) for odd i,
#   z = sqrt(-2 ln u1) (cos 2 pi u2 + j sin 2 pi u2) / sqrt(2)     (Box-Muller, CN(0, 1)).
PHILOX_M0, PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
PHILOX_W0, PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10 on uint32 counter arrays (numpy), returns four uint32 arrays."""
    c = [np.asarray(v, dtype=np.uint64) & _MASK32 for v in (c0, c1, c2, c3)]
    k0, k1 = np.uint64(k0 & 0xFFFFFFFF), np.uint64(k1 & 0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(PHILOX_M0) * c[0]
        p1 = np.uint64(PHILOX_M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + np.uint64(PHILOX_W0)) & _MASK32
        k1 = (k1 + np.uint64(PHILOX_W1)) & _MASK32
    return [v.astype(np.uint32) for v in c]


def ase_cn_philox(seed: int, block: int, span: int, n: int) -> np.ndarray:
    """CN(0,1) ASE draws [n] (complex128) of one (block, span), the generator the GPU kernel uses."""
    i = np.arange(n, dtype=np.uint64)
    m = i >> np.uint64(1)
    x0, x1, x2, x3 = philox4x32_10(m, np.full(n, span), np.full(n, block & 0xFFFFFFFF),
                                   np.full(n, (block >> 32) & 0xFFFFFFFF), seed & 0xFFFFFFFF,
                                   (seed >> 32) & 0xFFFFFFFF)
    odd = (i & np.uint64(1)).astype(bool)
    a = np.where(odd, x2, x0).astype(np.float64)
    b = np.where(odd, x3, x1).astype(np.float64)
    u1 = (a + 0.5) * 2.0 ** -32
    u2 = (b + 0.5) * 2.0 ** -32
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.exp(2j * np.pi * u2) / np.sqrt(2.0)
