"""Transmitter and fiber channel simulator (oracle; test infrastructure only).

Generates the seeded LDBP inputs the paper's way (§IV-A): periodic-frame RRC
shaping (Eq. 11), asymmetric split-step solution of the NLSE (Eqs. 4-6) with L_eff Kerr steps,
EDFA gain + ASE noise per span, brick-wall low-pass filter and sampling at rho_d samples/symbol.
Random draws (symbols, ASE) are inputs (from ldbp_inputs), never drawn here.
"""
from __future__ import annotations

import numpy as np

from . import physics


def rrc_response(n: int, sps: int, rolloff: float) -> np.ndarray:
    """Exact root-raised-cosine frequency response on the n-point DFT grid (reading G11).

    Frequencies in cycles/symbol f = fftfreq(n) * sps; RC(f) = 1 for |f| <= (1-b)/2,
    0.5 (1 + cos(pi/b (|f| - (1-b)/2))) up to (1+b)/2, 0 beyond; RRC = sqrt(RC)."""
    f = np.abs(np.fft.fftfreq(n) * sps)
    lo, hi = (1.0 - rolloff) / 2.0, (1.0 + rolloff) / 2.0
    rc = np.where(f <= lo, 1.0, np.where(f <= hi, 0.5 * (1.0 + np.cos(np.pi / rolloff * (f - lo))), 0.0))
    return np.sqrt(rc)


def modulate(symbols: np.ndarray, sps: int, power_w: float, rolloff: float = 0.1) -> np.ndarray:
    """x = sqrt(P) sum_k s_k p(t - k/R_s) on a periodic frame (Eq. 11).

    Implemented as circular convolution of the upsampled symbols with the RRC pulse; the
    factor sps makes the mean power P and the matched-filter output at symbol instants
    exactly sqrt(P) s_k (RRC^2 = RC is Nyquist)."""
    s = np.asarray(symbols, dtype=np.complex128)
    n = len(s) * sps
    z = np.zeros(n, dtype=np.complex128)
    z[::sps] = s
    return np.sqrt(power_w) * sps * np.fft.ifft(np.fft.fft(z) * rrc_response(n, sps, rolloff))


def kerr_step(u: np.ndarray, gamma: float, leff_km: float) -> np.ndarray:
    """sigma_z(u) = u e^{j gamma L_eff(z) |u|^2}."""
    return u * np.exp(1j * gamma * leff_km * np.abs(u) ** 2)


def linear_step(u: np.ndarray, z_km: float, alpha_np: float, beta2: float, fs_hz: float) -> np.ndarray:
    """A_z u = e^{-alpha z/2} F^{-1} diag(e^{z H_k}) F u, H_k = j beta2 omega_k^2 / 2."""
    w = physics.omega_grid(u.shape[-1], fs_hz)
    H = np.exp(-alpha_np * z_km / 2.0) * np.exp(1j * beta2 / 2.0 * w ** 2 * z_km)
    return np.fft.ifft(np.fft.fft(u) * H)


def ssfm(u: np.ndarray, deltas_km, alpha_np: float, beta2: float, gamma: float, fs_hz: float) -> np.ndarray:
    """Asymmetric split-step over consecutive segments (Eq. 6).

    Reading G5: each segment applies the L_eff Kerr step at its start, then the
    lossy linear step — the exact lumping of the loss that L_eff assumes."""
    for d in deltas_km:
        u = kerr_step(u, gamma, float(physics.l_eff(d, alpha_np)))
        u = linear_step(u, d, alpha_np, beta2, fs_hz)
    return u


def edfa(u: np.ndarray, alpha_np: float, span_km: float, psd_w_per_hz: float, fs_hz: float,
         noise_cn) -> np.ndarray:
    """Amplitude gain e^{alpha L_sp / 2} plus white circular Gaussian ASE with per-sample
    variance PSD * f_sim.  ``noise_cn`` are CN(0,1) draws or None."""
    out = u * np.exp(alpha_np * span_km / 2.0)
    if noise_cn is not None:
        out = out + np.sqrt(psd_w_per_hz * fs_hz) * noise_cn
    return out


def lowpass_decimate(u: np.ndarray, rho_a: int, rho_d: int) -> np.ndarray:
    """Ideal brick-wall LPF passing |f| <= f_s/2, f_s = rho_d R_s (reading G8), then sampling
    at t = k/f_s."""
    n = u.shape[-1]
    f = np.fft.fftfreq(n) * rho_a  # cycles per symbol
    U = np.fft.fft(u)
    U[np.abs(f) > rho_d / 2.0] = 0.0
    return np.fft.ifft(U)[:: rho_a // rho_d]


def simulate_link(symbols, power_w, *, num_spans, span_km, steps_per_span, alpha_db, beta2,
                  gamma, baud_hz, rho_a, rho_d, nf_db, nu_hz, ase_draws=None, rolloff=0.1,
                  adjust=0.4):
    """Full forward simulation of §IV-A: Tx at rho_a, N_sp x (SSFM span + EDFA), LPF, sample at rho_d.

    ``ase_draws``: list of N_sp CN(0,1) arrays of length N_sym*rho_a (or None: noiseless).
    Returns (r at rho_d, x_tx at rho_d)."""
    from .steps import log_step_sizes

    a = physics.alpha_np_per_km(alpha_db)
    fs_a = rho_a * baud_hz
    u = modulate(symbols, rho_a, power_w, rolloff)
    deltas = log_step_sizes(span_km, steps_per_span, a, adjust)
    psd = physics.ase_psd(nf_db, a, span_km, nu_hz)
    for k in range(num_spans):
        u = ssfm(u, deltas, a, beta2, gamma, fs_a)
        u = edfa(u, a, span_km, psd, fs_a, None if ase_draws is None else ase_draws[k])
    r = lowpass_decimate(u, rho_a, rho_d)
    x_tx = modulate(symbols, rho_d, power_w, rolloff)
    return r, x_tx
