"""Direct-form LDBP forward, adjoint, loss and Adam (oracle; test infrastructure only).

The model is Eq. (7): f_theta(x) = sigma_M(A^(M) ... sigma_1(A^(1) x)), where each
A^(i) is the circular convolution with a centred FIR filter h^(i) (reading G1:
a_t = sum_{j=-Kh}^{Kh} h_j u_{(t-j) mod n}, whose frequency response is the paper's DTFT
sum_k h_k e^{-jk omega}) and sigma_i(a) = a e^{j gamma'_i |a|^2} (P:384-388 with the
per-step scalar of Remark 2).  Everything here is evaluated literally, in
complex128, one step at a time: no blocking, fusion or reordering.

Gradient convention for a real loss L and complex z: g_z = dL/dRe z + j dL/dIm z, so
dL = Re(conj(g_z) dz).  The adjoint formulas are derived from Eq. (7)
and the chain rule; they are pinned by central finite differences and by the exact gauge
identities implied by Remark 4, see tests/test_oracle_ldbp.py.

Shapes: x, y, targets: complex128 [B][n]; taps: complex128 [M][T] (tap j at index j+Kh);
gamma: float64 [M].
"""
from __future__ import annotations

import numpy as np


def fir(u: np.ndarray, h: np.ndarray) -> np.ndarray:
    """Circular centred convolution a_t = sum_j h_j u_{(t-j) mod n} (reading G1)."""
    kh = (len(h) - 1) // 2
    a = np.zeros_like(u, dtype=np.complex128)
    for idx, j in enumerate(range(-kh, kh + 1)):
        a = a + h[idx] * np.roll(u, j, axis=-1)  # roll(u, j)[t] = u[t - j]
    return a


def kerr(a: np.ndarray, g: float) -> np.ndarray:
    """Pointwise Kerr rotation sigma(a) = a e^{j g |a|^2} (Remark 2 P:464-469)."""
    return a * np.exp(1j * g * np.abs(a) ** 2)


def forward(x: np.ndarray, taps: np.ndarray, gamma: np.ndarray, keep: bool = False):
    """LDBP forward pass, Eq. (7).  Returns y (and the per-step inputs u^(i-1), FIR outputs a^(i))."""
    u = np.asarray(x, dtype=np.complex128)
    us, as_ = [], []
    for i in range(len(gamma)):
        a = fir(u, np.asarray(taps[i], dtype=np.complex128))
        if keep:
            us.append(u)
            as_.append(a)
        u = kerr(a, float(gamma[i]))
    return (u, us, as_) if keep else u


def backward(x: np.ndarray, gy: np.ndarray, taps: np.ndarray, gamma: np.ndarray):
    """Reverse-mode sweep of Eq. (7) for an incoming gradient gy = dL/dy (convention above).

    Per step i = M..1, with p = |a|^2, phi = gamma'_i p, v = a e^{j phi}, gv = dL/dv:
      c_t   = Im(gv_t conj(v_t))
      ga_t  = gv_t e^{-j phi_t} + 2 gamma'_i c_t a_t
      dgamma'_i = sum_t c_t p_t
      dh_j  = sum_t ga_t conj(u_{t-j})            (u = u^(i-1), the FIR input)
      gu_s  = sum_j conj(h_j) ga_{s+j}
    Returns (dtaps complex [M][T], dgamma float [M], gx complex [B][n]); sums over the batch.
    """
    taps = np.asarray(taps, dtype=np.complex128)
    M, T = taps.shape
    kh = (T - 1) // 2
    _, us, as_ = forward(x, taps, gamma, keep=True)
    g = np.asarray(gy, dtype=np.complex128)
    dtaps = np.zeros((M, T), dtype=np.complex128)
    dgamma = np.zeros(M)
    for i in range(M - 1, -1, -1):
        a, u = as_[i], us[i]
        p = np.abs(a) ** 2
        phi = gamma[i] * p
        v = a * np.exp(1j * phi)
        c = np.imag(g * np.conj(v))
        ga = g * np.exp(-1j * phi) + 2.0 * gamma[i] * c * a
        dgamma[i] = np.sum(c * p)
        for idx, j in enumerate(range(-kh, kh + 1)):
            dtaps[i, idx] = np.sum(ga * np.conj(np.roll(u, j, axis=-1)))
        gu = np.zeros_like(ga)
        for idx, j in enumerate(range(-kh, kh + 1)):
            gu = gu + np.conj(taps[i, idx]) * np.roll(ga, -j, axis=-1)  # roll(ga,-j)[s] = ga[s+j]
        g = gu
    return dtaps, dgamma, g


def sym_fold(dtaps: np.ndarray) -> np.ndarray:
    """Gradient of the tied half parameters h_j = h_{-j}: g_j + g_{-j} at both positions."""
    T = dtaps.shape[-1]
    kh = (T - 1) // 2
    out = dtaps.copy()
    for j in range(1, kh + 1):
        s = dtaps[..., kh + j] + dtaps[..., kh - j]
        out[..., kh + j] = s
        out[..., kh - j] = s
    return out


def mse_sum(y: np.ndarray, target: np.ndarray) -> float:
    """Unscaled waveform squared error sum |y - x_tx|^2 (reading G7; Eq. (2) with the 1/N applied later)."""
    return float(np.sum(np.abs(y - target) ** 2))


def loss_grad(x, target, taps, gamma, mask=None, symmetric: bool = True):
    """The hot path's gradient buffer [sum|e|^2 | dgamma[M] | dtaps[M][T][2]] (fp64, UNscaled).

    Taps are multiplied by the binary mask before use; masked taps get gradient 0.
    With symmetric=True the tap gradient is the tied-parameter gradient (sym_fold).
    """
    taps = np.asarray(taps, dtype=np.complex128)
    M, T = taps.shape
    if mask is not None:
        taps = taps * np.asarray(mask, dtype=np.float64)
    y = forward(x, taps, gamma)
    loss = mse_sum(y, target)
    dtaps, dgamma, _ = backward(x, 2.0 * (y - target), taps, gamma)
    if symmetric:
        dtaps = sym_fold(dtaps)
    if mask is not None:
        dtaps = dtaps * np.asarray(mask, dtype=np.float64)
    buf = np.empty(1 + M + 2 * M * T)
    buf[0] = loss
    buf[1:1 + M] = dgamma
    buf[1 + M:] = np.stack([dtaps.real, dtaps.imag], axis=-1).reshape(-1)
    return buf


def pack_params(taps: np.ndarray, gamma: np.ndarray) -> np.ndarray:
    """Real parameter vector [Re/Im taps as [M][T][2] | gamma[M]] (Adam acts on reals)."""
    t = np.asarray(taps, dtype=np.complex128)
    return np.concatenate([np.stack([t.real, t.imag], axis=-1).reshape(-1), np.asarray(gamma, np.float64)])


def unpack_params(theta: np.ndarray, M: int, T: int):
    tr = theta[:2 * M * T].reshape(M, T, 2)
    return tr[..., 0] + 1j * tr[..., 1], theta[2 * M * T:].copy()


def grad_vector(buf: np.ndarray, M: int, T: int) -> np.ndarray:
    """Rearrange a loss_grad buffer into the pack_params order."""
    return np.concatenate([buf[1 + M:], buf[1:1 + M]])


def adam(theta, m, v, g, t: int, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, frozen=None):
    """Bias-corrected Adam (Kingma2015; paper P:810-812, mu = 1e-3 Table I; beta/eps
    defaults per reading G13).  ``frozen`` (bool array) keeps entries and their moments at 0
    change (masked taps are additionally forced to 0 by the caller).  Returns new (theta, m, v)."""
    theta = np.array(theta, dtype=np.float64)
    m = b1 * np.asarray(m, np.float64) + (1.0 - b1) * g
    v = b2 * np.asarray(v, np.float64) + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    step = lr * mh / (np.sqrt(vh) + eps)
    if frozen is not None:
        step = np.where(frozen, 0.0, step)
    return theta - step, m, v


def adam_update(buf, n_global, theta, m, v, t, M, T, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8,
                tap_mask=None, gamma_learnable=None):
    """The ABI's ldbp_adam_update semantics: g = buf/n_global (mean MSE gradient, Eq. (2));
    masked taps are forced to 0 with m = v = 0; non-learnable gamma' are frozen."""
    g = grad_vector(np.asarray(buf, np.float64), M, T) / float(n_global)
    frozen = np.zeros(2 * M * T + M, dtype=bool)
    tapmask_r = None
    if tap_mask is not None:
        tapmask_r = np.repeat(np.asarray(tap_mask, dtype=bool).reshape(-1), 2)
        frozen[:2 * M * T] = ~tapmask_r
    if gamma_learnable is not None:
        frozen[2 * M * T:] = ~np.asarray(gamma_learnable, dtype=bool)
    theta, m, v = adam(theta, m, v, np.where(frozen, 0.0, g), t, lr, b1, b2, eps, frozen)
    if tapmask_r is not None:
        theta[:2 * M * T] = np.where(tapmask_r, theta[:2 * M * T], 0.0)
        m[:2 * M * T] = np.where(tapmask_r, m[:2 * M * T], 0.0)
        v[:2 * M * T] = np.where(tapmask_r, v[:2 * M * T], 0.0)
    return theta, m, v


def scale_gauge(taps, gamma, i: int, c: complex):
    """Remark 4 exact reparameterisation: (h^(i)/c, gamma'_i |c|^2, c h^(i+1)).

    Since |a/c|^2 |c|^2 = |a|^2 the Kerr phase is unchanged, sigma_i's output is scaled by 1/c
    and the next filter undoes it; f_theta is unchanged for every input."""
    t = np.array(taps, dtype=np.complex128)
    g = np.array(gamma, dtype=np.float64)
    t[i] = t[i] / c
    g[i] = g[i] * abs(c) ** 2
    t[i + 1] = t[i + 1] * c
    return t, g
