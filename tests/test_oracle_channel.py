"""Pins for oracle.channel and oracle.receiver: soliton, energy conservation, Nyquist RRC
chain, genie phase, effective SNR and the DBP limit on a simulated link."""
import numpy as np
import pytest

import ldbp_inputs as li
from oracle import channel, ldbp, physics, receiver, steps


def test_fundamental_soliton_first_order_convergence():
    """alpha = 0, noiseless: u(0,t) = sqrt(P0) sech(t/T0), P0 = |beta2|/(gamma T0^2) is an exact
    NLSE solution u(z,t) = u(0,t) e^{j gamma P0 z / 2} (Eq. 4).  The asymmetric SSM
    error must shrink ~2x when the step count doubles (O(1/M))."""
    beta2 = physics.ps2_per_km(-21.7)
    gamma = 1.3
    T0 = 20e-12
    P0 = abs(beta2) / (gamma * T0 ** 2)
    n = 1024
    dt = T0 / 16
    t = (np.arange(n) - n // 2) * dt
    u0 = np.sqrt(P0) / np.cosh(t / T0)
    L = 2 * T0 ** 2 / abs(beta2)
    exact = u0 * np.exp(1j * gamma * P0 * L / 2)
    errs = []
    for M in (16, 32, 64):
        u = channel.ssfm(u0.astype(complex), [L / M] * M, 0.0, beta2, gamma, 1 / dt)
        errs.append(np.linalg.norm(u - exact) / np.linalg.norm(exact))
    assert errs[-1] < 2e-2
    for e1, e2 in zip(errs[:-1], errs[1:]):
        assert 1.6 <= e1 / e2 <= 2.4, errs


def test_lossless_energy_conservation():
    """alpha = 0 noiseless: every SSM factor is unitary or a pure phase."""
    u = li.cn(np.random.default_rng(1), 512) * 0.05
    out = channel.ssfm(u, [10.0, 20.0, 50.0], 0.0, physics.ps2_per_km(-21.7), 1.3, 42.8e9)
    assert abs(np.linalg.norm(out) / np.linalg.norm(u) - 1) < 1e-12
    # linear steps compose exactly: A_{z1} A_{z2} = A_{z1+z2}
    a = channel.linear_step(channel.linear_step(u, 30.0, 0.01, -2e-23, 42.8e9), 50.0, 0.01, -2e-23, 42.8e9)
    b = channel.linear_step(u, 80.0, 0.01, -2e-23, 42.8e9)
    np.testing.assert_allclose(a, b, atol=1e-14)


def test_rrc_chain_recovers_symbols_exactly():
    """modulate -> matched filter -> downsample gives s exactly (RRC^2 Nyquist on a periodic
    frame); mean power is P; SNR = 1/MSE for one frame."""
    s = li.qam16(li.rng(0, 0, "symbols"), 512)
    for sps in (2, 4):
        P = 1e-3
        x = channel.modulate(s, sps, P)
        st = receiver.matched_filter_downsample(x, sps, P)
        np.testing.assert_allclose(st, s, atol=1e-12)
    x = channel.modulate(li.cn(np.random.default_rng(2), 4096), 2, 2e-3)
    assert abs(np.mean(np.abs(x) ** 2) / 2e-3 - 1) < 0.05
    # decimating a band-limited rho_a waveform equals generating it at rho_d
    xa = channel.modulate(s, 4, 1e-3)
    xd = channel.lowpass_decimate(xa, 4, 2)
    np.testing.assert_allclose(xd, channel.modulate(s, 2, 1e-3), atol=1e-15 + 1e-12 * np.abs(xd).max())
    e = 0.1 * li.cn(np.random.default_rng(3), 512)
    pooled, literal = receiver.effective_snr_db([(s + e, s)])
    mse = np.mean(np.abs(e) ** 2)
    assert abs(pooled - 10 * np.log10(1 / mse)) < 1e-12 and abs(pooled - literal) < 1e-12


def test_genie_phase():
    s = li.qam16(li.rng(0, 1, "symbols"), 256)
    for phi in (0.3, -2.0, np.pi - 1e-3):
        sh, ph = receiver.genie_phase(s * np.exp(1j * phi), s)
        assert abs(np.angle(np.exp(1j * (ph - phi)))) < 1e-12
        np.testing.assert_allclose(sh, s, atol=1e-12)
    # phi_hat minimises the error over a 1-D scan
    st = s * np.exp(0.4j) + 0.3 * li.cn(np.random.default_rng(4), 256)
    sh, ph = receiver.genie_phase(st, s)
    base = np.sum(np.abs(sh - s) ** 2)
    for d in (-0.01, 0.01):
        assert np.sum(np.abs(st * np.exp(-1j * (ph + d)) - s) ** 2) >= base


LINK = dict(span_km=80.0, alpha_db=0.2, beta2=physics.ps2_per_km(-21.7), gamma=1.3, baud_hz=10.7e9,
            rho_a=4, rho_d=2, nf_db=5.0, nu_hz=1.946e14)


def _ldbp_full_taps(n, deltas, fs, beta2):
    """Full-length exact inverse-CD taps per step (T = n+1, halved +-n/2), direct from the DFT."""
    w = physics.omega_grid(n, fs)
    j = np.arange(-n // 2, n // 2 + 1)
    E = np.exp(2j * np.pi * np.outer(j, np.arange(n)) / n) / n
    taps = []
    for d in deltas:
        h = E @ np.exp(-1j * beta2 / 2 * w ** 2 * d)
        h[0] *= 0.5
        h[-1] *= 0.5
        taps.append(h)
    return np.array(taps)


def test_dbp_limit_and_sign():
    """P4: a -30 dBm noiseless link through LDBP with full-length inverse-CD taps recovers the
    symbols (>40 dB).  At high power, DBP with gamma' of G3/G4 beats linear-only and the
    opposite-sign nonlinearity (pins the DBP sign reading G3)."""
    nsym, spans = 256, 3
    s = li.qam16(li.rng(0, 0, "symbols"), nsym)
    fs = LINK["rho_d"] * LINK["baud_hz"]
    deltas, gam = steps.dbp_plan(spans, 80.0, 1, 0.2, 1.3)
    taps = _ldbp_full_taps(nsym * 2, deltas, fs, LINK["beta2"])
    snrs = {}
    for pdbm in (-30.0, 8.0):
        P = physics.dbm_to_w(pdbm)
        r, x_tx = channel.simulate_link(s, P, num_spans=spans, steps_per_span=20, **LINK)
        for name, g in (("dbp", gam), ("lin", 0 * gam), ("neg", -gam)):
            y = ldbp.forward(r[None], taps, g)[0]
            snrs[(pdbm, name)] = receiver.evaluate([y], [s], [P])[0]
    assert snrs[(-30.0, "dbp")] > 40.0
    assert snrs[(8.0, "dbp")] > snrs[(8.0, "lin")] + 3.0 > snrs[(8.0, "neg")] + 3.0


def test_ase_noise_variance():
    """Per-sample ASE variance PSD * f_sim from CN(0,1) draws."""
    a = physics.alpha_np_per_km(0.2)
    psd = physics.ase_psd(5.0, a, 80.0, 1.946e14)
    w = li.cn(np.random.default_rng(7), 200000)
    out = channel.edfa(np.zeros(200000, complex), a, 80.0, psd, 42.8e9, w)
    assert abs(np.mean(np.abs(out) ** 2) / (psd * 42.8e9) - 1) < 0.02
    u = np.ones(4, complex)
    np.testing.assert_allclose(np.abs(channel.edfa(u, a, 80.0, psd, 42.8e9, None)) ** 2, np.exp(a * 80.0))


def test_rx_fir_matched_filter_pins():
    """The truncated-FIR matched filter (reading G19) agrees with the exact frequency-domain RRC
    matched filter to the truncation error, keeps the Nyquist property (RRC^2 at symbol instants
    = delta) and its adjoint is the transpose (<M y, g> = <y, M^T g>)."""
    s = li.qam16(li.rng(0, 3, "symbols"), 512)
    for sps in (2, 4):
        h = receiver.rrc_fir_taps(sps, 0.1, 32)
        assert len(h) == 2 * 32 * sps + 1
        np.testing.assert_allclose(h, h[::-1], atol=1e-15)
        x = channel.modulate(s, sps, 1.0)
        st = receiver.mf_fir_downsample(x, h, sps)
        assert np.max(np.abs(st - s)) < 2e-3  # 10% roll-off tails beyond 32 symbols
        # exact FIR (full circular response) reproduces the frequency-domain MF to 1e-12
        n = len(x)
        hfull = np.fft.ifft(channel.rrc_response(n, sps, 0.1)).real
        # lags -n/2..n/2; +-n/2 alias to the same circular lag, so each carries half its weight
        hfull = np.concatenate([hfull[-(n // 2):], hfull[: n // 2 + 1]])
        hfull[0] *= 0.5
        hfull[-1] *= 0.5
        np.testing.assert_allclose(receiver.mf_fir_downsample(x, hfull, sps), s, atol=1e-10)
    rng = np.random.default_rng(8)
    y = rng.standard_normal((2, 96)) + 1j * rng.standard_normal((2, 96))
    g = rng.standard_normal((2, 48)) + 1j * rng.standard_normal((2, 48))
    h = receiver.rrc_fir_taps(2, 0.1, 8)
    lhs = np.sum(np.conj(g) * receiver.mf_fir_downsample(y, h, 2))
    rhs = np.sum(np.conj(receiver.mf_fir_adjoint(g, h, 2, 96)) * y)
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)


def test_rx_loss_gradient_finite_differences():
    """Symbol-MSE loss after MF + genie phase (Eq. (12)-(13)): the chain-rule gradient w.r.t. the
    LDBP output matches central differences; dL/dphi vanishes at the genie phase (it minimises
    the error over phi), so the phase path contributes nothing."""
    rng = np.random.default_rng(9)
    n, sps = 64, 2
    h = receiver.rrc_fir_taps(sps, 0.1, 4)
    y = (rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))) * 0.1
    s = li.qam16(li.rng(0, 4, "symbols"), n).reshape(2, n // 2)
    P = np.array([1e-2, 2e-2])
    errs, gy, dphi = receiver.rx_loss_grad(y, s, P, h, sps)
    assert np.all(np.abs(dphi) < 1e-12 * np.abs(errs).max())
    eps = 1e-6
    scale = np.abs(gy).max()
    for b, t in [(0, 0), (0, 7), (1, 63), (1, 30)]:
        for u in (1.0, 1j):
            yp, ym = y.copy(), y.copy()
            yp[b, t] += eps * u
            ym[b, t] -= eps * u
            fd = (receiver.rx_loss(yp, s, P, h, sps)[0].sum() - receiver.rx_loss(ym, s, P, h, sps)[0].sum()) / (2 * eps)
            an = gy[b, t].real if u == 1.0 else gy[b, t].imag
            assert abs(fd - an) <= 1e-6 * scale


# ---- exact circulant matched filter (NEXT-1, Eq. (12)) ----
def test_exact_mf_recovers_symbols_and_is_zero_loss():
    """Nyquist pin (P11): modulate -> exact circulant MF -> downsample returns s exactly, so the
    receiver-chain loss of the transmitted waveform itself is 0 (any power, any phase)."""
    from oracle import receiver

    s = li.qam16(li.rng(81, 0, "symbols"), 512)
    for sps in (2, 4):
        x = channel.modulate(s, sps, 2e-3) * np.exp(0.7j)
        errs, gy = receiver.rx_loss_grad_exact(x, s, [2e-3], sps)
        assert errs[0] < 1e-20 * len(s)
        assert np.max(np.abs(gy)) < 1e-9


def test_exact_mf_adjoint_identity():
    """Re<M y, g> = Re<y, M^T g> for random y, g (the adjoint used by the gradient)."""
    from oracle import receiver

    g0 = np.random.default_rng(3)
    for n, sps in ((1024, 2), (512, 4), (96, 1)):
        y = g0.standard_normal(n) + 1j * g0.standard_normal(n)
        g = g0.standard_normal(n // sps) + 1j * g0.standard_normal(n // sps)
        lhs = np.real(np.vdot(g, receiver.mf_exact(y, sps)))
        rhs = np.real(np.vdot(receiver.mf_exact_adjoint(g, sps, n), y))
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_exact_rx_loss_finite_differences_and_weights():
    """Central finite differences of L = sum_b w_b errs_b w.r.t. Re / Im of sampled y entries
    match dL/dy (gradient convention dL/dRe + j dL/dIm), including the genie-phase path."""
    from oracle import receiver

    B, nsym, sps = 2, 64, 2
    s = np.stack([li.qam16(li.rng(82, b, "symbols"), nsym) for b in range(B)])
    y = np.stack([channel.modulate(s[b], sps, 1e-3) for b in range(B)])
    y = y + 1e-3 * (li.cn(li.rng(82, 9, "ase"), y.shape))  # noisy: non-zero loss and gradient
    pw, w = [1e-3, 1e-3], np.array([0.7, 1.9])
    errs, gy = receiver.rx_loss_grad_exact(y, s, pw, sps, weights=w)
    L = lambda yy: float(np.sum(w * receiver.rx_loss_grad_exact(yy, s, pw, sps)[0]))  # noqa: E731
    h = 1e-8
    for b, t in ((0, 3), (1, 50), (0, 127)):
        for unit in (1.0, 1j):
            yp, ym = y.copy(), y.copy()
            yp[b, t] += h * unit
            ym[b, t] -= h * unit
            fd = (L(yp) - L(ym)) / (2 * h)
            an = gy[b, t].real if unit == 1.0 else gy[b, t].imag
            assert abs(fd - an) <= 1e-5 * np.max(np.abs(gy)) + 1e-6 * abs(an), (b, t, unit, fd, an)
    # weights scale each block's gradient, not its (unweighted) error
    errs1, gy1 = receiver.rx_loss_grad_exact(y, s, pw, sps)
    np.testing.assert_allclose(errs, errs1, rtol=1e-14)
    np.testing.assert_allclose(gy[1], w[1] * gy1[1], rtol=1e-12, atol=1e-18)


def test_truncated_fir_converges_to_exact_mf():
    """The round-1 truncated FIR (reading G19) approaches the exact circulant as its span grows."""
    from oracle import receiver

    s = li.qam16(li.rng(83, 0, "symbols"), 2048)
    y = channel.modulate(s, 2, 1.0) + 0.1 * li.cn(li.rng(83, 1, "ase"), 4096)
    ex = receiver.mf_exact(y, 2)
    errs = [np.max(np.abs(receiver.mf_fir_downsample(y, receiver.rrc_fir_taps(2, span_symbols=sp), 2) - ex))
            for sp in (8, 32, 256)]
    assert errs[0] > errs[1] > errs[2]
