"""Step sizes and parameter initialisation (oracle; test infrastructure only).

Paper §IV-C: logarithmic step sizes (Zhang2013c, adjusting factor 0.4), half-step
merging (Example 1), least-squares filter initialisation, pruning masks.
"""
from __future__ import annotations

import numpy as np

from . import physics


def log_step_sizes(span_km: float, steps_per_span: int, alpha_np: float, adjust: float = 0.4) -> np.ndarray:
    """Per-span step sizes in FORWARD order (small steps first, where power is high).

    The paper only cites the heuristic ("logarithmic heuristic in [Zhang2013c] ...
    adjusting factor 0.4"); SPEC S:297-305 restates it: with alpha' = adjust*alpha, boundary
    z_k satisfies 1 - e^{-alpha' z_k} = (k/M)(1 - e^{-alpha' L_sp}).  Pinned by Example 1
    (P:872-883): L_sp = 100 km, 2 StPS -> (~30, ~70) km.
    """
    a = adjust * alpha_np
    m = steps_per_span
    if a == 0.0:
        return np.full(m, span_km / m)
    k = np.arange(m + 1)
    z = -np.log(1.0 - (k / m) * (1.0 - np.exp(-a * span_km))) / a
    z[-1] = span_km
    return np.diff(z)


def merge_half_steps(deltas) -> np.ndarray:
    """Symmetric SSM half-step merging (Example 1): (d1/2, (d1+d2)/2, ..., dM/2)."""
    d = np.asarray(deltas, dtype=np.float64)
    out = np.empty(len(d) + 1)
    out[0] = d[0] / 2.0
    out[1:-1] = (d[:-1] + d[1:]) / 2.0
    out[-1] = d[-1] / 2.0
    return out


def xi_of(delta_km: float, beta2_s2_per_km: float, fs_hz: float) -> float:
    """xi = -beta2 delta' f_s^2 / 2 (Table I)."""
    return -beta2_s2_per_km * delta_km * fs_hz ** 2 / 2.0


def ls_taps(xi: float, taps: int, n_grid: int = 512, band: float | None = None,
            oob_weight: float = 1e-2, cap: float | None = None) -> np.ndarray:
    """Least-squares FIR fit of the inverse-CD response d(omega) = e^{j xi omega^2}.

    min_h || B h - d ||^2 with B_{i,k} = e^{-j k omega_i} (the paper's DTFT),
    k = -Kh..Kh, on the uniform grid omega_i = 2 pi i / N, i = -N/2 .. N/2-1 (reading G12:
    the paper's i = -N/2..N/2 would count omega = +-pi twice).  With ``band`` (fraction of
    f_s, e.g. 0.275 for 10% RRC at 2 sps) the out-of-band rows are down-weighted by
    ``oob_weight`` — a simplified stand-in for the constrained design of Sheikh2016, which
    the paper does not reproduce (parity unpinned for the weighted variant; full-band is
    pinned against the closed-form truncated IDFT).  With ``cap`` the filter is then scaled
    so that max_w |F(h)(w)| <= cap on a dense grid (reading G12b: a stand-in for the paper's
    out-of-band gain constraint, with SPEC's default cap 1.0; it makes every step
    non-expansive so short filters cannot inflate the signal power over many steps).
    Returns complex128 [T], index j+Kh.
    """
    kh = (taps - 1) // 2
    i = np.arange(-n_grid // 2, n_grid // 2)
    w = 2.0 * np.pi * i / n_grid
    k = np.arange(-kh, kh + 1)
    B = np.exp(-1j * np.outer(w, k))
    d = np.exp(1j * xi * w ** 2)
    if band is not None:
        wt = np.where(np.abs(w) <= 2.0 * np.pi * band, 1.0, oob_weight)
        B = B * wt[:, None]
        d = d * wt
    h, *_ = np.linalg.lstsq(B, d, rcond=None)
    if cap is not None:
        wd = np.linspace(-np.pi, np.pi, 8193)
        gain = np.abs(np.exp(-1j * np.outer(wd, k)) @ h).max()
        if gain > cap:
            h = h * (cap / gain)
    return h


def gamma_prime(gamma_per_w_km: float, alpha_np: float, z_start_km: float, delta_km: float) -> float:
    """DBP nonlinear scalar for the step that inverts forward segment [z_a, z_a+delta].

    Reading G3/G4: gamma' = -gamma * e^{-alpha z_a} * L_eff(delta) — the sign
    inverts the Kerr phase (P:1041 sigma_i = sigma_{delta_i}; DBP sign implicit in the paper),
    e^{-alpha z_a} is the launch-normalised power at the segment start (all-pass LS filters keep
    the signal at launch level), L_eff per P:399-400.  Parity unpinned beyond the closed form
    -gamma L_eff(L_sp) at 1 StPS (the kernel takes gamma' as an input).
    """
    return -gamma_per_w_km * np.exp(-alpha_np * z_start_km) * float(physics.l_eff(delta_km, alpha_np))


def dbp_plan(num_spans: int, span_km: float, steps_per_span: int, alpha_db: float,
             gamma_per_w_km: float, adjust: float = 0.4):
    """Asymmetric-SSM DBP plan (l = M): per model step (delta_i, gamma'_i) in
    processing order (last forward segment of the last span first)."""
    a = physics.alpha_np_per_km(alpha_db)
    fwd = log_step_sizes(span_km, steps_per_span, a, adjust)
    starts = np.concatenate([[0.0], np.cumsum(fwd)[:-1]])
    deltas, gammas = [], []
    for _ in range(num_spans):
        for d, z0 in zip(fwd[::-1], starts[::-1]):
            deltas.append(d)
            gammas.append(gamma_prime(gamma_per_w_km, a, z0, d))
    return np.array(deltas), np.array(gammas)


def unit_taps(steps: int, taps: int) -> np.ndarray:
    """Unit (identity) filters h = delta_0."""
    h = np.zeros((steps, taps), dtype=np.complex128)
    h[:, (taps - 1) // 2] = 1.0
    return h


def total_impulse_length(tap_lengths) -> int:
    """Length of the filter obtained by convolving all sub-filters: sum(T_i - 1) + 1."""
    return int(sum(int(t) - 1 for t in tap_lengths) + 1)


def pruning_events(initial_lengths, target_lengths) -> int:
    """Number of pruning steps; each removes the two outermost taps of one filter."""
    return int(sum((int(a) - int(b)) // 2 for a, b in zip(initial_lengths, target_lengths)))


def prune_mask(taps: int, target: int) -> np.ndarray:
    """Binary mask keeping the central `target` taps of a length-`taps` symmetric filter."""
    kh, kt = (taps - 1) // 2, (target - 1) // 2
    m = np.zeros(taps, dtype=np.uint8)
    m[kh - kt: kh + kt + 1] = 1
    return m
