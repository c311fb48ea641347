"""Pins for oracle.ldbp: the FIR orientation (paper DTFT), finite differences, Remark-4 gauge
invariants, delay-tap closed form, equivariance, masks and Adam closed forms."""
import numpy as np
import pytest

import ldbp_inputs as li
from oracle import channel, ldbp, physics


def rnd(shape, seed, scale=1.0):
    g = np.random.default_rng(seed)
    return (g.standard_normal(shape) + 1j * g.standard_normal(shape)) * scale


def test_fir_frequency_response_is_paper_dtft():
    """Applied to e^{j w t}, the filter returns F(h)(w) e^{j w t} with the paper's DTFT
    F(h) = sum_k h_k e^{-j k w}.  Non-symmetric taps, so a transposed or
    shifted convolution fails."""
    n = 64
    h = rnd(7, 1)
    t = np.arange(n)
    for m in (0, 1, 5, 31, 32, 50):
        w = 2 * np.pi * m / n
        u = np.exp(1j * w * t)
        H = np.sum(h * np.exp(-1j * np.arange(-3, 4) * w))
        np.testing.assert_allclose(ldbp.fir(u, h), H * u, atol=1e-12)


def test_fir_equals_circulant_matrix_product():
    """A^(i) x with the circulant A_{t,s} = h_{(t-s) wrapped}, brute force."""
    n, T = 11, 5
    h = rnd(T, 2)
    x = rnd(n, 3)
    A = np.zeros((n, n), complex)
    for t in range(n):
        for j in range(-2, 3):
            A[t, (t - j) % n] += h[j + 2]
    np.testing.assert_allclose(ldbp.fir(x, h), A @ x, atol=1e-13)
    # T > n wraps several times: still the periodic-extension convolution
    h9 = rnd(9, 4)
    x3 = rnd(3, 5)
    A3 = np.zeros((3, 3), complex)
    for t in range(3):
        for j in range(-4, 5):
            A3[t, (t - j) % 3] += h9[j + 4]
    np.testing.assert_allclose(ldbp.fir(x3, h9), A3 @ x3, atol=1e-13)


def test_kerr_preserves_modulus_and_delta_zero_is_identity():
    """|sigma(x)_t| = |x_t|; gamma' = 0 (delta = 0) is the identity."""
    x = rnd((3, 40), 6)
    y = ldbp.kerr(x, -13.0)
    np.testing.assert_allclose(np.abs(y), np.abs(x), rtol=1e-14)
    np.testing.assert_array_equal(ldbp.kerr(x, 0.0), x)


def _loss(x, tgt, taps, gamma):
    return ldbp.mse_sum(ldbp.forward(x, taps, gamma), tgt)


@pytest.mark.parametrize("seed,M,T,n,B", [(0, 3, 5, 32, 2), (1, 4, 3, 40, 1), (2, 2, 7, 33, 2), (3, 1, 1, 16, 1)])
def test_adjoint_matches_central_finite_differences(seed, M, T, n, B):
    """Every tap, gamma' and input gradient vs central differences."""
    x = rnd((B, n), 10 + seed, 0.7)
    tgt = rnd((B, n), 20 + seed, 0.7)
    taps = rnd((M, T), 30 + seed, 0.3)
    taps[:, (T - 1) // 2] += 1.0
    gamma = np.random.default_rng(40 + seed).uniform(-1.5, 1.5, M)
    y = ldbp.forward(x, taps, gamma)
    dt, dg, gx = ldbp.backward(x, 2 * (y - tgt), taps, gamma)
    eps = 1e-6
    scale = max(np.abs(dt).max(), np.abs(dg).max())
    for i in range(M):
        for k in range(T):
            for comp, unit in ((0, 1.0), (1, 1j)):
                tp, tm = taps.copy(), taps.copy()
                tp[i, k] += eps * unit
                tm[i, k] -= eps * unit
                fd = (_loss(x, tgt, tp, gamma) - _loss(x, tgt, tm, gamma)) / (2 * eps)
                an = dt[i, k].real if comp == 0 else dt[i, k].imag
                assert abs(fd - an) <= 1e-5 * scale, (i, k, comp, fd, an)
        gp, gm = gamma.copy(), gamma.copy()
        gp[i] += eps
        gm[i] -= eps
        fd = (_loss(x, tgt, taps, gp) - _loss(x, tgt, taps, gm)) / (2 * eps)
        assert abs(fd - dg[i]) <= 1e-5 * scale, (i, fd, dg[i])
    gsc = np.abs(gx).max()
    for (b, t) in [(0, 0), (0, n // 2), (B - 1, n - 1)]:
        for unit in (1.0, 1j):
            xp, xm = x.copy(), x.copy()
            xp[b, t] += eps * unit
            xm[b, t] -= eps * unit
            fd = (_loss(xp, tgt, taps, gamma) - _loss(xm, tgt, taps, gamma)) / (2 * eps)
            an = gx[b, t].real if unit == 1.0 else gx[b, t].imag
            assert abs(fd - an) <= 1e-5 * gsc


def test_sym_fold_is_tied_parameter_gradient():
    """With h_{-j} = h_j tied the gradient of h_j is g_j + g_{-j}: check by FD on the tie."""
    M, T, n = 2, 5, 24
    x = rnd((1, n), 50, 0.8)
    tgt = rnd((1, n), 51, 0.8)
    half = rnd((M, 3), 52, 0.3)
    half[:, 0] += 1
    taps = np.concatenate([half[:, :0:-1], half], axis=1)
    gamma = np.array([0.7, -1.1])
    buf = ldbp.loss_grad(x, tgt, taps, gamma, symmetric=True)
    dt = buf[1 + M:].reshape(M, T, 2)
    eps = 1e-6
    for i in range(M):
        for j in range(3):
            hp, hm = half.copy(), half.copy()
            hp[i, j] += eps
            hm[i, j] -= eps
            tp = np.concatenate([hp[:, :0:-1], hp], axis=1)
            tm = np.concatenate([hm[:, :0:-1], hm], axis=1)
            fd = (_loss(x, tgt, tp, gamma) - _loss(x, tgt, tm, gamma)) / (2 * eps)
            assert abs(fd - dt[i, 2 + j, 0]) < 1e-6 * np.abs(dt).max()
            assert dt[i, 2 + j, 0] == dt[i, 2 - j, 0]


def test_forward_gauge_invariance_remark4():
    """Remark 4: (h^(i)/c, gamma'_i|c|^2, c h^(i+1)) leaves f_theta unchanged."""
    M, T, n = 4, 5, 48
    x = rnd((2, n), 60, 0.6)
    taps = rnd((M, T), 61, 0.3)
    taps[:, 2] += 1
    gamma = np.array([-0.8, 0.5, -1.2, 0.9])
    y = ldbp.forward(x, taps, gamma)
    for i, c in [(0, 1.7), (1, 0.4 * np.exp(0.9j)), (2, np.exp(-2.1j))]:
        t2, g2 = ldbp.scale_gauge(taps, gamma, i, c)
        np.testing.assert_allclose(ldbp.forward(x, t2, g2), y, atol=1e-12)


def test_gradient_gauge_identities():
    """Differentiating the Remark-4 invariance, for 1 <= i < M:
    Re<g_{i+1},h_{i+1}> - Re<g_i,h_i> + 2 gamma'_i g_{gamma'_i} = 0 and
    Im<g_i,h_i> = Im<g_{i+1},h_{i+1}>, with <g,h> = sum conj(g) h."""
    M, T, n = 5, 7, 40
    x = rnd((2, n), 70, 0.6)
    tgt = rnd((2, n), 71, 0.6)
    taps = rnd((M, T), 72, 0.3)
    taps[:, 3] += 1
    gamma = np.random.default_rng(73).uniform(-1, 1, M)
    y = ldbp.forward(x, taps, gamma)
    dt, dg, _ = ldbp.backward(x, 2 * (y - tgt), taps, gamma)
    ip = [np.sum(np.conj(dt[i]) * taps[i]) for i in range(M)]
    mag = max(abs(v) for v in ip)
    for i in range(M - 1):
        assert abs(ip[i + 1].real - ip[i].real + 2 * gamma[i] * dg[i]) < 1e-12 * mag
        assert abs(ip[i].imag - ip[i + 1].imag) < 1e-12 * mag


def test_delay_taps_closed_form():
    """h^(i) = e^{j theta_i} delta_{j_i}: y_t = x_{t-S} exp(j(sum theta + sum gamma' |x_{t-S}|^2)),
    S = sum j_i (delay taps keep |.| so every Kerr phase sees |x|^2)."""
    n, T = 37, 7
    shifts = [2, -3, 1, 3]
    th = [0.3, -1.2, 2.0, 0.1]
    gamma = np.array([0.5, -0.7, 1.1, -0.2])
    taps = np.zeros((4, T), complex)
    for i, (j, t) in enumerate(zip(shifts, th)):
        taps[i, j + 3] = np.exp(1j * t)
    x = rnd((2, n), 80, 0.9)
    y = ldbp.forward(x, taps, gamma)
    xs = np.roll(x, sum(shifts), axis=-1)
    ref = xs * np.exp(1j * (sum(th) + gamma.sum() * np.abs(xs) ** 2))
    np.testing.assert_allclose(y, ref, atol=1e-13)


def test_shift_phase_equivariance():
    """f(shift_k(e^{j phi} x)) = shift_k(e^{j phi} f(x)) (circular, phase-blind Kerr)."""
    x = rnd((1, 50), 90)
    taps = rnd((3, 5), 91, 0.3)
    taps[:, 2] += 1
    gamma = np.array([0.4, -0.9, 0.6])
    y = ldbp.forward(x, taps, gamma)
    for k, phi in [(7, 0.5), (-13, -2.0)]:
        y2 = ldbp.forward(np.roll(np.exp(1j * phi) * x, k, axis=-1), taps, gamma)
        np.testing.assert_allclose(y2, np.roll(np.exp(1j * phi) * y, k, axis=-1), atol=1e-12)


def test_linear_inverse_full_length_taps():
    """gamma = 0, noiseless: the full-length inverse-CD filter (T = n+1, +-n/2 taps halved)
    in the direct-form LDBP reproduces the channel input exactly."""
    n = 64
    fs = 21.4e9
    beta2 = physics.ps2_per_km(-21.7)
    x = rnd(n, 100)
    z = 160.0
    r = channel.linear_step(x, z, 0.0, beta2, fs)
    w = physics.omega_grid(n, fs)
    D = np.exp(-1j * beta2 / 2 * w ** 2 * z)
    j = np.arange(-n // 2, n // 2 + 1)
    h = np.array([np.sum(D * np.exp(2j * np.pi * np.arange(n) * jj / n)) / n for jj in j])
    h[0] *= 0.5
    h[-1] *= 0.5
    np.testing.assert_allclose(h, h[::-1], atol=1e-12)
    y = ldbp.forward(r[None], h[None], np.zeros(1))
    np.testing.assert_allclose(y[0], x, atol=1e-10 * np.abs(x).max())


def test_masked_taps_zero_gradient():
    M, T, n = 3, 7, 30
    x = rnd((1, n), 110, 0.7)
    tgt = rnd((1, n), 111, 0.7)
    taps = rnd((M, T), 112, 0.3)
    taps[:, 3] += 1
    mask = np.ones((M, T), np.uint8)
    mask[0, [0, 6]] = 0
    mask[2, [0, 1, 5, 6]] = 0
    buf = ldbp.loss_grad(x, tgt, taps, np.array([0.3, -0.4, 0.5]), mask=mask, symmetric=False)
    dt = buf[1 + M:].reshape(M, T, 2)
    assert np.all(dt[mask == 0] == 0)
    assert np.all(np.abs(dt[mask == 1]).sum(-1) > 0)
    # masked forward == forward with the masked taps set to zero
    tz = taps * mask
    np.testing.assert_allclose(
        buf[0], ldbp.mse_sum(ldbp.forward(x, tz, np.array([0.3, -0.4, 0.5])), tgt), rtol=1e-14)


def test_adam_closed_forms():
    """Bias-corrected Adam: with a constant gradient g the update is exactly lr*g/(|g|+eps)
    at every t (m_hat = g, v_hat = g^2), so the first step is ~mu ([0.999mu, mu]);
    zero gradient leaves parameters unchanged."""
    lr = 1e-3
    theta = np.array([0.5, -0.2, 3.0, 0.0])
    g = np.array([2.0, -1e-3, 0.0, 1e-7])
    m = np.zeros(4)
    v = np.zeros(4)
    th = theta.copy()
    for t in range(1, 6):
        th_new, m, v = ldbp.adam(th, m, v, g, t, lr=lr)
        step = th - th_new
        np.testing.assert_allclose(step, lr * g / (np.abs(g) + 1e-8), rtol=1e-9, atol=1e-18)
        th = th_new
    first = np.abs(lr * g[[0, 1]] / (np.abs(g[[0, 1]]) + 1e-8))
    assert np.all(first <= lr) and np.all(first >= 0.999 * lr)
    assert th[2] == theta[2]


def test_adam_update_mask_and_frozen_gamma():
    M, T = 2, 3
    theta = ldbp.pack_params(np.ones((M, T)) * (0.5 + 0.1j), np.array([-1.0, -2.0]))
    buf = np.arange(1 + M + 2 * M * T, dtype=float) + 1.0
    mask = np.array([[0, 1, 0], [1, 1, 1]], np.uint8)
    th, m, v = ldbp.adam_update(buf, 10.0, theta, np.zeros_like(theta), np.zeros_like(theta), 1, M, T,
                                tap_mask=mask, gamma_learnable=np.array([1, 0], np.uint8))
    t_new, g_new = ldbp.unpack_params(th, M, T)
    assert t_new[0, 0] == 0 and t_new[0, 2] == 0 and m[0] == 0 and v[0] == 0
    assert g_new[1] == -2.0 and g_new[0] != -1.0
    assert np.all(t_new[1] != 0.5 + 0.1j)


def test_inputs_are_independent_of_rank_count():
    """Blocks are keyed by global index: any sharding reproduces the same union (§8(e))."""
    full = li.gaussian_blocks(3, range(8), 16, 1e-3)
    part = np.concatenate([li.gaussian_blocks(3, range(r * 2, r * 2 + 2), 16, 1e-3) for r in range(4)])
    np.testing.assert_array_equal(full, part)
    s = li.qam16(li.rng(0, 0, "symbols"), 4096)
    assert abs(np.mean(np.abs(s) ** 2) - 1.0) < 0.05
    assert set(np.round(np.unique(s.real) * np.sqrt(10), 12)) == {-3.0, -1.0, 1.0, 3.0}
