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
