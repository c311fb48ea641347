"""Receiver DSP after LDBP and the figure of merit (oracle; test infrastructure only).

s_hat = e^{-j phi} M f_theta(r) (Eq. 12): RRC matched filter + downsampling (the
circulant M), genie phase phi = arg(s^H s_tilde), effective SNR (Eq. 14,
P:829-835).  Reading G10: s_tilde is divided by sqrt(P) before the comparison with unit-power
symbols.  Reading G9: the primary SNR is pooled 1/MSE; the literal mean-of-inverses is also
returned.
"""
from __future__ import annotations

import numpy as np

from .channel import rrc_response


def matched_filter_downsample(y: np.ndarray, sps: int, power_w: float, rolloff: float = 0.1) -> np.ndarray:
    """s_tilde = (RRC matched filter of y)[::sps] / sqrt(P)."""
    n = y.shape[-1]
    z = np.fft.ifft(np.fft.fft(y) * rrc_response(n, sps, rolloff))
    return z[..., ::sps] / np.sqrt(power_w)


def genie_phase(s_tilde: np.ndarray, s: np.ndarray):
    """phi_hat = arg(s^H s_tilde), s_hat = s_tilde e^{-j phi_hat}."""
    phi = np.angle(np.sum(np.conj(s) * s_tilde))
    return s_tilde * np.exp(-1j * phi), phi


def effective_snr_db(frames):
    """frames: list of (s_hat, s).  Returns (pooled SNR dB, mean-of-inverses SNR dB) (Eq. 14)."""
    errs = np.array([np.sum(np.abs(sh - s) ** 2) for sh, s in frames])
    nsym = len(frames[0][1])
    pooled = nsym * len(frames) / np.sum(errs)
    literal = nsym * np.mean(1.0 / errs)
    return 10.0 * np.log10(pooled), 10.0 * np.log10(literal)


def evaluate(y_blocks, symbols_blocks, powers_w, sps: int = 2, rolloff: float = 0.1):
    """Per-block receiver chain, returns (pooled dB, literal dB) over the given blocks."""
    frames = []
    for y, s, p in zip(y_blocks, symbols_blocks, powers_w):
        st = matched_filter_downsample(np.asarray(y, np.complex128), sps, p, rolloff)
        sh, _ = genie_phase(st, s)
        frames.append((sh, s))
    return effective_snr_db(frames)


# ---------------------------------------------------------------------------------------------
# Receiver-chain training loss: symbol MSE after the matched filter,
# downsampling and genie phase correction (Eq. (12), loss P:812-816, Eq. (13)).
# Reading G19: on the GPU the circulant M is a decimating circular FIR whose taps are
# the exact periodic RRC impulse response truncated to +-span symbols; the oracle uses the same
# definition so parity is exact, and pins the taps against the exact frequency-domain RRC.
# ---------------------------------------------------------------------------------------------
def rrc_fir_taps(sps: int, rolloff: float = 0.1, span_symbols: int = 32, n_ref: int = 1 << 18) -> np.ndarray:
    """Real, even taps h[m], m = -span*sps..span*sps: the impulse response of the frequency-domain
    RRC (rrc_response) on a long circular grid n_ref (alias-free to ~1e-12), truncated."""
    H = rrc_response(n_ref, sps, rolloff)
    h = np.fft.ifft(H).real
    L = span_symbols * sps
    return np.concatenate([h[-L:], h[:L + 1]])


def mf_fir_downsample(y: np.ndarray, h: np.ndarray, sps: int) -> np.ndarray:
    """s_tilde_k = sum_m h[m] y_{(k sps - m) mod n} (circular decimating FIR = the circulant M)."""
    y = np.asarray(y, np.complex128)
    n = y.shape[-1]
    Lh = (len(h) - 1) // 2
    k = np.arange(n // sps) * sps
    out = np.zeros(y.shape[:-1] + (n // sps,), np.complex128)
    for idx, m in enumerate(range(-Lh, Lh + 1)):
        out = out + h[idx] * y[..., (k - m) % n]
    return out


def mf_fir_adjoint(g: np.ndarray, h: np.ndarray, sps: int, n: int) -> np.ndarray:
    """M^T (h real): g_y[t] = sum_k sum_m h[m] [k sps - m == t mod n] g_k, per block."""
    g = np.atleast_2d(np.asarray(g, np.complex128))
    Lh = (len(h) - 1) // 2
    out = np.zeros((g.shape[0], n), np.complex128)
    k = np.arange(g.shape[-1]) * sps
    for idx, m in enumerate(range(-Lh, Lh + 1)):
        for b in range(g.shape[0]):
            np.add.at(out[b], (k - m) % n, h[idx] * g[b])
    return out


def rx_loss(y, s, power_w, h, sps):
    """Per-block symbol error energy sum_k |s_hat - s|^2 with s_hat = e^{-j phi} M y / sqrt(P),
    phi = arg(s^H M y) (genie).  Returns (errs [B], s_tilde, phi)."""
    st = mf_fir_downsample(y, h, sps)
    s = np.asarray(s, np.complex128)
    z = np.sum(np.conj(s) * st, axis=-1)
    phi = np.angle(z)
    a = np.exp(-1j * phi) / np.sqrt(np.asarray(power_w, np.float64))
    e = a[..., None] * st - s
    return np.sum(np.abs(e) ** 2, axis=-1), st, phi


def rx_loss_grad(y, s, power_w, h, sps):
    """dL/dy of L = sum_blocks errs, by the full chain rule through the genie phase phi(s_tilde)
    (no envelope shortcut): g_st = 2 conj(a) e + (dL/dphi) j s / conj(z), then g_y = M^T g_st."""
    y = np.asarray(y, np.complex128)
    errs, st, phi = rx_loss(y, s, power_w, h, sps)
    s = np.asarray(s, np.complex128)
    z = np.sum(np.conj(s) * st, axis=-1)
    a = np.exp(-1j * phi) / np.sqrt(np.asarray(power_w, np.float64))
    sh = a[..., None] * st
    e = sh - s
    g_direct = 2.0 * np.conj(a)[..., None] * e
    dL_dphi = 2.0 * np.sum(np.real(np.conj(e) * (-1j) * sh), axis=-1)  # d s_hat / d phi = -j s_hat
    g_phi = 1j * s / np.conj(z)[..., None]  # d phi = Im(conj(z) dz)/|z|^2, z = s^H s_tilde
    g_st = g_direct + dL_dphi[..., None] * g_phi
    gy = mf_fir_adjoint(g_st, h, sps, y.shape[-1]).reshape(y.shape)
    return errs, gy, dL_dphi


# ---------------------------------------------------------------------------------------------
# Exact circulant matched filter (Eq. (12): "M ... a circulant matrix that represents
# the matched filter"): M y = (F^-1 diag(RRC) F y)[::sps].  C = F^-1 diag(RRC) F is real and
# symmetric (RRC real and even in frequency), so M^T g = C U g with U the zero-stuffing upsampler.
# This is the definition itself; the truncated-FIR form above is its approximation (reading G19).
# ---------------------------------------------------------------------------------------------
def mf_exact(y: np.ndarray, sps: int, rolloff: float = 0.1) -> np.ndarray:
    """s_tilde = M y (unnormalised), exact circulant RRC matched filter then downsampling."""
    y = np.asarray(y, np.complex128)
    n = y.shape[-1]
    return np.fft.ifft(np.fft.fft(y, axis=-1) * rrc_response(n, sps, rolloff), axis=-1)[..., ::sps]


def mf_exact_adjoint(g: np.ndarray, sps: int, n: int, rolloff: float = 0.1) -> np.ndarray:
    """M^T g = C U g (zero-stuff the symbol-rate gradient, then the same circulant)."""
    g = np.asarray(g, np.complex128)
    u = np.zeros(g.shape[:-1] + (n,), np.complex128)
    u[..., ::sps] = g
    return np.fft.ifft(np.fft.fft(u, axis=-1) * rrc_response(n, sps, rolloff), axis=-1)


def rx_loss_grad_exact(y, s, power_w, sps: int, rolloff: float = 0.1, weights=None):
    """L = sum_b w_b errs_b with the exact M (Eq. (12)-(13)); returns (errs [B] unweighted, dL/dy).
    Same chain rule as rx_loss_grad (genie phase included), with M and M^T exact."""
    y = np.atleast_2d(np.asarray(y, np.complex128))
    s = np.atleast_2d(np.asarray(s, np.complex128))
    B, n = y.shape
    w = np.ones(B) if weights is None else np.asarray(weights, np.float64)
    st = mf_exact(y, sps, rolloff)
    z = np.sum(np.conj(s) * st, axis=-1)
    phi = np.angle(z)
    a = np.exp(-1j * phi) / np.sqrt(np.asarray(power_w, np.float64))
    sh = a[:, None] * st
    e = sh - s
    errs = np.sum(np.abs(e) ** 2, axis=-1)
    g_direct = 2.0 * np.conj(a)[:, None] * e
    dL_dphi = 2.0 * np.sum(np.real(np.conj(e) * (-1j) * sh), axis=-1)
    g_st = w[:, None] * (g_direct + dL_dphi[:, None] * (1j * s / np.conj(z)[:, None]))
    return errs, mf_exact_adjoint(g_st, sps, n, rolloff)
