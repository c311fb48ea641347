"""Learned enhanced SSM (ESSM): LDBP with filtered nonlinear steps (oracle; test infrastructure).

Paper §III-D, Eq. (nl_filtered): every nonlinear step filters the squared modulus
before the phase rotation,
    [sigma^(i)(a)]_t = a_t exp(j gamma'_i sum_{k=-kappa}^{kappa} eta^(i)_k |a_{(t-k) mod n}|^2),
with real per-step filters eta^(i) (2 kappa + 1 taps, tap k at index k + kappa); the linear
steps are the FIRs of Eq. (7) (oracle.ldbp.fir).  gamma'_i carries gamma L_eff of the paper's
step (reading G20: kept as a separate scalar so kappa = 0, eta = [1] is exactly
Eq. (7)).  Parameters: theta = {h^(i), eta^(i), gamma'_i}.

Evaluated literally in complex128, one step at a time.  Gradient convention as oracle.ldbp
(g_z = dL/dRe z + j dL/dIm z).  The adjoint (chain rule) per step, with p = |a|^2,
psi = eta (*) p (psi_t = sum_k eta_k p_{t-k}), phi = gamma' psi, v = a e^{j phi}, gv = dL/dv:
    c_t    = Im(gv_t conj(v_t))                    (= dL/dphi_t)
    q_m    = gamma' sum_k eta_k c_{m+k}            (= dL/dp_m)
    ga_t   = gv_t e^{-j phi_t} + 2 q_t a_t
    dgamma' = sum_t c_t psi_t,   deta_k = gamma' sum_t c_t p_{t-k}
    dh_j   = sum_t ga_t conj(u_{t-j}),   gu_s = sum_j conj(h_j) ga_{s+j}
Pinned in tests/test_oracle_essm.py (kappa = 0 reduces to oracle.ldbp exactly; central finite
differences on every parameter and on the input; |v| = |a|; shifted-delta filter closed form).
"""
from __future__ import annotations

import numpy as np

from .ldbp import fir


def shift(p: np.ndarray, k: int) -> np.ndarray:
    """s_t = p_{(t-k) mod n}."""
    return np.roll(p, k, axis=-1)


def filt(p: np.ndarray, eta: np.ndarray) -> np.ndarray:
    """psi_t = sum_k eta_k p_{(t-k) mod n}, k = -kappa..kappa (eta[k + kappa])."""
    kap = (len(eta) - 1) // 2
    out = np.zeros(p.shape, dtype=np.float64)
    for idx, k in enumerate(range(-kap, kap + 1)):
        out = out + float(eta[idx]) * shift(p, k)
    return out


def nl(a: np.ndarray, g: float, eta: np.ndarray) -> np.ndarray:
    """Filtered nonlinear step, Eq. (nl_filtered)."""
    return a * np.exp(1j * g * filt(np.abs(a) ** 2, eta))


def forward(x, taps, gamma, eta, keep: bool = False):
    """ESSM forward: u <- nl(fir(u, h^(i)), gamma'_i, eta^(i)), i = 1..M."""
    u = np.asarray(x, dtype=np.complex128)
    us = []
    for i in range(len(gamma)):
        if keep:
            us.append(u)
        a = fir(u, np.asarray(taps[i], dtype=np.complex128))
        u = nl(a, float(gamma[i]), np.asarray(eta[i], dtype=np.float64))
    return (u, us) if keep else u


def backward(x, gy, taps, gamma, eta):
    """Reverse sweep for gy = dL/dy.  Returns (dtaps complex [M][T], dgamma [M], deta [M][2kappa+1],
    gx); parameter gradients summed over the batch."""
    taps = np.asarray(taps, dtype=np.complex128)
    eta = np.asarray(eta, dtype=np.float64)
    M, T = taps.shape
    kh = (T - 1) // 2
    kap = (eta.shape[1] - 1) // 2
    _, us = forward(x, taps, gamma, eta, keep=True)
    g = np.asarray(gy, dtype=np.complex128)
    dtaps = np.zeros((M, T), np.complex128)
    dgamma = np.zeros(M)
    deta = np.zeros(eta.shape)
    for i in reversed(range(M)):
        u = us[i]
        a = fir(u, taps[i])
        p = np.abs(a) ** 2
        psi = filt(p, eta[i])
        phi = gamma[i] * psi
        v = a * np.exp(1j * phi)
        c = np.imag(g * np.conj(v))
        q = np.zeros(c.shape)
        for idx, k in enumerate(range(-kap, kap + 1)):
            q = q + eta[i][idx] * shift(c, -k)  # c_{m+k}
        q = gamma[i] * q
        ga = g * np.exp(-1j * phi) + 2.0 * q * a
        dgamma[i] = np.sum(c * psi)
        for idx, k in enumerate(range(-kap, kap + 1)):
            deta[i][idx] = gamma[i] * np.sum(c * shift(p, k))
        gu = np.zeros_like(u)
        for idx, j in enumerate(range(-kh, kh + 1)):
            dtaps[i, idx] = np.sum(ga * np.conj(shift(u, j)))
            gu = gu + np.conj(taps[i, idx]) * shift(ga, -j)  # ga_{s+j}
        g = gu
    return dtaps, dgamma, deta, g


def loss_grad(x, target, taps, gamma, eta, symmetric: bool = True):
    """[sum|y - target|^2 | dgamma [M] | dtaps [M][T][2] | deta [M][2kappa+1]] for the waveform
    MSE (reading G7), unscaled; symmetric: tied taps h_{-j} = h_j (oracle.ldbp.sym_fold)."""
    from .ldbp import sym_fold

    y = forward(x, taps, gamma, eta)
    e = y - np.asarray(target, dtype=np.complex128)
    dt, dg, de, _ = backward(x, 2.0 * e, taps, gamma, eta)
    if symmetric:
        dt = sym_fold(dt)
    return np.concatenate([[np.sum(np.abs(e) ** 2)], dg, np.stack([dt.real, dt.imag], -1).reshape(-1),
                           np.asarray(de).reshape(-1)])
