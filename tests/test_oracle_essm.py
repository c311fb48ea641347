"""Pins of the ESSM oracle (oracle/essm.py, Eq. nl_filtered), CPU only."""
import numpy as np

import ldbp_inputs as li
from oracle import essm, ldbp as O


def rand_model(seed, M, T, kap, sym=True):
    taps = li.random_sym_taps(seed, M, T, 0.1) if sym else li.random_general_taps(seed, M, T, 0.1)
    gamma = li.random_gamma(seed, M, -3.0, -0.5)
    g = np.random.default_rng(seed)
    eta = g.uniform(-0.5, 1.0, (M, 2 * kap + 1))
    return taps, gamma, eta


def test_kappa0_is_ldbp():
    """kappa = 0, eta = [1]: Eq. (nl_filtered) is the standard nonlinear step, so ESSM = Eq. (7)
    for the forward and every gradient (dgamma, dtaps); deta_0 = gamma' dgamma' by the chain rule."""
    x = li.gaussian_blocks(1, range(2), 64, 1.0)
    taps, gamma, _ = rand_model(1, 3, 5, 0)
    eta = np.ones((3, 1))
    np.testing.assert_allclose(essm.forward(x, taps, gamma, eta), O.forward(x, taps, gamma), rtol=0, atol=1e-13)
    gy = li.gaussian_blocks(1, range(2), 64, 1.0, purpose="grad")
    dt, dg, de, gx = essm.backward(x, gy, taps, gamma, eta)
    rdt, rdg, rgx = O.backward(x, gy, taps, gamma)
    np.testing.assert_allclose(dt, rdt, atol=1e-11)
    np.testing.assert_allclose(dg, rdg, atol=1e-11)
    np.testing.assert_allclose(gx, rgx, atol=1e-11)
    np.testing.assert_allclose(de[:, 0], gamma * dg, atol=1e-11)


def test_phase_only_and_delta_filter():
    """|sigma(a)| = |a| (phase-only step); with eta = delta at k0 the phase at t is
    gamma' |a_{t-k0}|^2 (modulo-n indexing), a closed form."""
    rng = np.random.default_rng(2)
    a = rng.standard_normal((2, 40)) + 1j * rng.standard_normal((2, 40))
    eta = rng.uniform(-1, 1, 7)
    v = essm.nl(a, 0.7, eta)
    np.testing.assert_allclose(np.abs(v), np.abs(a), rtol=1e-14)
    for k0 in (-3, 0, 2):
        e = np.zeros(7)
        e[k0 + 3] = 1.0
        v = essm.nl(a, 0.7, e)
        t = np.arange(40)
        expect = a * np.exp(1j * 0.7 * np.abs(a[:, (t - k0) % 40]) ** 2)
        np.testing.assert_allclose(v, expect, rtol=1e-14)


def test_finite_differences_all_parameters():
    """Central differences of L = sum |y - target|^2 w.r.t. every tap (re, im), gamma', every
    eta tap and input samples, kappa > Kh and a filter wider than half the block (wraps)."""
    B, n, M, T, kap = 2, 24, 3, 5, 4
    x = li.gaussian_blocks(3, range(B), n, 1.0)
    tgt = li.gaussian_blocks(3, range(B), n, 1.0, purpose="target")
    taps, gamma, eta = rand_model(3, M, T, kap, sym=False)

    def L(xx, tt, gg, ee):
        return np.sum(np.abs(essm.forward(xx, tt, gg, ee) - tgt) ** 2)

    y = essm.forward(x, taps, gamma, eta)
    dt, dg, de, gx = essm.backward(x, 2 * (y - tgt), taps, gamma, eta)
    eps = 1e-6
    checks = []
    for i in range(M):
        for idx in (0, 2, 4):
            for u in (1.0, 1j):
                tp, tm = taps.copy(), taps.copy()
                tp[i, idx] += eps * u
                tm[i, idx] -= eps * u
                fd = (L(x, tp, gamma, eta) - L(x, tm, gamma, eta)) / (2 * eps)
                checks.append((fd, dt[i, idx].real if u == 1.0 else dt[i, idx].imag))
        gp, gm = gamma.copy(), gamma.copy()
        gp[i] += eps
        gm[i] -= eps
        checks.append(((L(x, taps, gp, eta) - L(x, taps, gm, eta)) / (2 * eps), dg[i]))
        for k in (0, kap, 2 * kap):
            ep, em = eta.copy(), eta.copy()
            ep[i, k] += eps
            em[i, k] -= eps
            checks.append(((L(x, taps, gamma, ep) - L(x, taps, gamma, em)) / (2 * eps), de[i, k]))
    for b, t in ((0, 0), (1, 17)):
        for u in (1.0, 1j):
            xp, xm = x.copy(), x.copy()
            xp[b, t] += eps * u
            xm[b, t] -= eps * u
            fd = (L(xp, taps, gamma, eta) - L(xm, taps, gamma, eta)) / (2 * eps)
            checks.append((fd, gx[b, t].real if u == 1.0 else gx[b, t].imag))
    fd, an = np.array(checks).T
    scale = np.abs(an).max()
    assert np.max(np.abs(fd - an)) <= 1e-5 * scale, np.max(np.abs(fd - an)) / scale


def test_loss_grad_layout_and_symmetric_fold():
    """buf = [loss | dgamma | dtaps re/im | deta]; the symmetric form ties +-j (oracle.ldbp.sym_fold)."""
    B, n, M, T, kap = 2, 32, 2, 5, 2
    x = li.gaussian_blocks(4, range(B), n, 1.0)
    tgt = li.gaussian_blocks(4, range(B), n, 1.0, purpose="target")
    taps, gamma, eta = rand_model(4, M, T, kap)
    buf = essm.loss_grad(x, tgt, taps, gamma, eta, symmetric=True)
    assert buf.shape == (1 + M + 2 * M * T + M * (2 * kap + 1),)
    y = essm.forward(x, taps, gamma, eta)
    assert np.isclose(buf[0], np.sum(np.abs(y - tgt) ** 2))
    dt, dg, de, _ = essm.backward(x, 2 * (y - tgt), taps, gamma, eta)
    np.testing.assert_allclose(buf[1:1 + M], dg)
    np.testing.assert_allclose(buf[1 + M + 2 * M * T:].reshape(M, -1), de)
    dts = buf[1 + M:1 + M + 2 * M * T].reshape(M, T, 2)
    np.testing.assert_allclose(dts[:, 1, 0], (dt[:, 1] + dt[:, 3]).real)
