"""Physical units and closed-form link quantities (oracle; test infrastructure only).

All lengths in km, times in s, powers in W, beta2 in s^2/km, gamma in 1/(W km).
"""
from __future__ import annotations

import numpy as np

PLANCK = 6.626e-34  # J s, Table I


def alpha_np_per_km(alpha_db_per_km: float) -> float:
    """dB/km -> nepers (power) per km: alpha = alpha_dB * ln(10)/10 (Table I)."""
    return alpha_db_per_km * np.log(10.0) / 10.0


def l_eff(z_km, alpha_np: float):
    """Effective nonlinear length L_eff(z) = (1 - e^{-alpha z})/alpha; -> z as alpha->0."""
    z = np.asarray(z_km, dtype=np.float64)
    if alpha_np == 0.0:
        return z
    return (1.0 - np.exp(-alpha_np * z)) / alpha_np


def n_sp(nf_db: float, alpha_np: float, span_km: float) -> float:
    """Spontaneous emission factor n_sp = N_F (2 (1 - e^{-alpha L_sp}))^{-1}."""
    nf = 10.0 ** (nf_db / 10.0)
    return nf / (2.0 * (1.0 - np.exp(-alpha_np * span_km)))


def ase_psd(nf_db: float, alpha_np: float, span_km: float, nu_hz: float) -> float:
    """EDFA noise PSD (e^{alpha L_sp} - 1) h nu_s n_sp in W/Hz."""
    return (np.exp(alpha_np * span_km) - 1.0) * PLANCK * nu_hz * n_sp(nf_db, alpha_np, span_km)


def t_cd(beta2_s2_per_km: float, delta_f_hz: float, length_km: float, fs_hz: float) -> float:
    """CD memory in samples, Eq. (15): T_cd = 2 pi |beta2| Delta_f L f_s."""
    return 2.0 * np.pi * abs(beta2_s2_per_km) * delta_f_hz * length_km * fs_hz


def ps2_per_km(beta2_ps2_per_km: float) -> float:
    """ps^2/km -> s^2/km."""
    return beta2_ps2_per_km * 1e-24


def dbm_to_w(p_dbm):
    return 10.0 ** ((np.asarray(p_dbm, dtype=np.float64) - 30.0) / 10.0)


def omega_grid(n: int, fs_hz: float) -> np.ndarray:
    """DFT angular frequencies omega_k = 2 pi f_k in rad/s, numpy fftfreq order.

    Reading G2: the paper's 1-based rule is off by one at k = n/2; we use the
    0-based convention m < n/2 -> m/n, else (m - n)/n.  Only the Nyquist bin differs, where
    omega^2 is the same either way.
    """
    m = np.arange(n)
    f = np.where(m < n / 2, m / n, (m - n) / n) * fs_hz
    return 2.0 * np.pi * f
