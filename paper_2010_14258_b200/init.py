"""Host-side parameter initialisation for LDBP (product helper, not on the hot path).

Independent of oracle/ (which has its own implementation; tests compare the two):
  - step sizes from the logarithmic heuristic with adjusting factor 0.4 (Example 1)
  - DBP nonlinear scalars gamma' (reading G3/G4 in DESIGN.md)
  - least-squares-truncated inverse-CD taps: on a uniform full-band grid the LS
    solution is the centred truncated inverse DTFT of e^{j xi w^2}, computed here in closed form.
"""
from __future__ import annotations

import math

import numpy as np


def alpha_nepers(alpha_db_per_km: float) -> float:
    return alpha_db_per_km * math.log(10.0) / 10.0


def leff(z_km: float, a: float) -> float:
    return z_km if a == 0 else -math.expm1(-a * z_km) / a


def span_steps(span_km: float, steps: int, alpha_db_per_km: float, adjust: float = 0.4) -> np.ndarray:
    """Forward-order step sizes of one span (equal shares of 1 - e^{-adjust*alpha*z})."""
    a = adjust * alpha_nepers(alpha_db_per_km)
    if a == 0:
        return np.full(steps, span_km / steps)
    total = -math.expm1(-a * span_km)
    bounds = [-math.log1p(-total * k / steps) / a for k in range(steps + 1)]
    bounds[-1] = span_km
    return np.diff(np.array(bounds))


def dbp_schedule(num_spans: int, span_km: float, steps_per_span: int, alpha_db_per_km: float = 0.2,
                 gamma_per_w_km: float = 1.3, adjust: float = 0.4):
    """Per model step (delta_i km, gamma'_i 1/W), processing order: spans and segments reversed."""
    a = alpha_nepers(alpha_db_per_km)
    fwd = span_steps(span_km, steps_per_span, alpha_db_per_km, adjust)
    z0 = np.concatenate(([0.0], np.cumsum(fwd)[:-1]))
    d_one = fwd[::-1]
    g_one = np.array([-gamma_per_w_km * math.exp(-a * z) * leff(d, a) for d, z in zip(fwd[::-1], z0[::-1])])
    return np.tile(d_one, num_spans), np.tile(g_one, num_spans)


def inverse_cd_taps(delta_km: float, taps: int, beta2_ps2_per_km: float = -21.7, fs_hz: float = 21.4e9,
                    grid: int = 512, cap: float | None = 1.0) -> np.ndarray:
    """Symmetric complex taps h_{-K..K} (index j+K) fitting e^{j xi w^2}, xi = -beta2 delta f_s^2 / 2.

    With ``cap`` (default 1.0) the fit is scaled so that its gain never exceeds ``cap`` at any
    frequency (a non-expansive stand-in for the out-of-band gain constraint of P:905-907)."""
    xi = -(beta2_ps2_per_km * 1e-24) * delta_km * fs_hz ** 2 / 2.0
    K = (taps - 1) // 2
    w = 2.0 * np.pi * (np.arange(grid) - grid // 2) / grid
    resp = np.exp(1j * xi * w * w)
    # centred inverse DTFT: h_k = (1/N) sum_i d(w_i) e^{j k w_i}; d is even so h_k = h_{-k}
    ks = np.arange(-K, K + 1)
    h = (resp[None, :] * np.exp(1j * ks[:, None] * w[None, :])).mean(axis=1)
    if cap is not None:
        dense = np.linspace(-np.pi, np.pi, 8193)
        peak = float(np.max(np.abs(np.exp(-1j * dense[:, None] * ks[None, :]) @ h)))
        h = h * min(1.0, cap / peak)
    return h


def model_taps(deltas_km, taps: int, **kw) -> np.ndarray:
    return np.stack([inverse_cd_taps(float(d), taps, **kw) for d in deltas_km])


def random_taps(rng: np.random.Generator, steps: int, taps: int) -> np.ndarray:
    """Random init of §V-E: iid N(0,1) re/im, then h <- h / sum_j |h_j|^2."""
    h = rng.standard_normal((steps, taps)) + 1j * rng.standard_normal((steps, taps))
    return h / np.sum(np.abs(h) ** 2, axis=1, keepdims=True)
