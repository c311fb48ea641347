"""Pins for oracle.physics and oracle.steps against the paper's worked examples and closed forms."""
import json
import os

import numpy as np
import pytest

from oracle import physics, steps


def test_example1_log_steps_and_merge(golden_dir):
    """Example 1: 2 x 100 km, 2 StPS -> (70, 30, 70, 30) km, merged (35, 50, 50, 50, 15)."""
    g = json.load(open(os.path.join(golden_dir, "example1_steps.json")))
    a = physics.alpha_np_per_km(g["alpha_db_per_km"])
    fwd = steps.log_step_sizes(g["span_km"], g["steps_per_span"], a, g["adjust"])
    dbp = np.tile(fwd[::-1], g["num_spans"])
    np.testing.assert_allclose(dbp, g["expected_dbp_order_km"], atol=g["tol_km"])
    merged = steps.merge_half_steps(dbp)
    np.testing.assert_allclose(merged, g["expected_merged_km"], atol=g["tol_km"])
    # partition property: the steps tile the span exactly
    assert abs(fwd.sum() - g["span_km"]) < 1e-9
    assert abs(merged.sum() - dbp.sum()) < 1e-9


def test_log_steps_limits():
    a = physics.alpha_np_per_km(0.2)
    assert np.allclose(steps.log_step_sizes(80.0, 1, a), [80.0])
    # adjust -> 0 approaches uniform steps (continuity of the heuristic)
    np.testing.assert_allclose(steps.log_step_sizes(80.0, 4, a, adjust=1e-9), 20.0, rtol=1e-6)
    # forward order: strictly increasing step sizes (small steps where the power is high)
    d = steps.log_step_sizes(80.0, 4, a)
    assert np.all(np.diff(d) > 0)


def test_tcd_golden(golden_dir):
    """Eq. (15): T_cd ~ 69 and 307."""
    g = json.load(open(os.path.join(golden_dir, "tcd.json")))
    b2 = physics.ps2_per_km(g["beta2_ps2_per_km"])
    for c in g["cases"]:
        t = physics.t_cd(b2, c["delta_f_hz"], c["length_km"], c["fs_hz"])
        assert abs(t - c["expected"]) <= c["tol"], (t, c)


def test_leff_closed_forms():
    a = physics.alpha_np_per_km(0.2)
    # alpha -> 0 limit is z; small-z expansion z - alpha z^2/2
    assert physics.l_eff(80.0, 0.0) == 80.0
    z = 1e-3
    assert abs(physics.l_eff(z, a) - (z - a * z * z / 2)) < 1e-12
    # infinite-length limit 1/alpha
    assert abs(physics.l_eff(1e6, a) - 1.0 / a) < 1e-9
    # 80 km SMF (SURVEY Appendix A recomputation): 21.169 km
    assert abs(physics.l_eff(80.0, a) - 21.169) < 1e-3


def test_ase_psd_formula():
    """PSD = (e^{aL}-1) h nu n_sp with n_sp = NF/(2(1-e^{-aL})): reduces to
    NF h nu e^{aL}/2 analytically; SPEC S:155 quotes 8.12e-18 W/Hz for 80 km, NF 5 dB."""
    a = physics.alpha_np_per_km(0.2)
    psd = physics.ase_psd(5.0, a, 80.0, 1.946e14)
    closed = 10 ** 0.5 * physics.PLANCK * 1.946e14 * np.exp(a * 80.0) / 2.0
    assert abs(psd - closed) / closed < 1e-12
    assert abs(psd - 8.12e-18) / 8.12e-18 < 5e-3


def test_total_taps_and_pruning(golden_dir):
    """77 total taps and 10 pruning events (Example 2)."""
    g = json.load(open(os.path.join(golden_dir, "taps_counts.json")))
    assert steps.total_impulse_length(g["tap_lengths"]) == g["expected_total"]
    # independent check: the convolution of the sub-filters has that length
    rng = np.random.default_rng(0)
    h = np.array([1.0 + 0j])
    for t in g["tap_lengths"]:
        h = np.convolve(h, rng.standard_normal(t) + 1j * rng.standard_normal(t))
    assert len(h) == g["expected_total"]
    assert steps.pruning_events(g["initial_lengths"], g["target_lengths"]) == g["expected_events"]
    m = steps.prune_mask(9, 7)
    assert list(m) == [0, 1, 1, 1, 1, 1, 1, 1, 0]


def test_ls_taps_closed_form_and_specials():
    """Full-band LS on a uniform grid = truncated centred inverse DFT (column orthogonality);
    delta' = 0 gives the unit filter; the fit is exactly symmetric."""
    N = 256
    for T in (3, 5, 9, 15):
        kh = (T - 1) // 2
        xi = steps.xi_of(80.0, physics.ps2_per_km(-21.7), 21.4e9)
        h = steps.ls_taps(xi, T, n_grid=N)
        i = np.arange(-N // 2, N // 2)
        w = 2 * np.pi * i / N
        d = np.exp(1j * xi * w ** 2)
        closed = np.array([np.sum(d * np.exp(1j * k * w)) / N for k in range(-kh, kh + 1)])
        np.testing.assert_allclose(h, closed, atol=1e-12)
        np.testing.assert_allclose(h, h[::-1], atol=1e-12)
        h0 = steps.ls_taps(0.0, T, n_grid=N)
        ref = np.zeros(T, complex)
        ref[kh] = 1
        np.testing.assert_allclose(h0, ref, atol=1e-12)
    # xi for one 80 km span at 21.4 GHz: 0.397 rad
    assert abs(steps.xi_of(80.0, physics.ps2_per_km(-21.7), 21.4e9) - 0.397) < 1e-3


def test_gamma_prime_closed_forms():
    """1 StPS: gamma' = -gamma L_eff(80 km) = -27.52 /W (P:399-400 with P:1041)."""
    a = physics.alpha_np_per_km(0.2)
    d, g = steps.dbp_plan(25, 80.0, 1, 0.2, 1.3)
    assert len(d) == 25 and np.allclose(d, 80.0)
    assert np.allclose(g, -1.3 * physics.l_eff(80.0, a))
    assert abs(g[0] + 27.52) < 5e-3
    # several steps per span: e^{-a z_a} L_eff(delta) = int_{z_a}^{z_a+delta} e^{-a z} dz, so the
    # per-span nonlinear-phase budget is partitioned exactly: sum gamma'_i = -gamma L_eff(L_sp).
    for spans in (2, 4):
        d2, g2 = steps.dbp_plan(1, 80.0, spans, 0.2, 1.3)
        assert abs(d2.sum() - 80.0) < 1e-9
        assert np.all(np.diff(d2) < 0)  # DBP order: largest step first
        assert abs(g2.sum() + 1.3 * physics.l_eff(80.0, a)) < 1e-12
        assert np.all(np.abs(g2) < 1.3 * physics.l_eff(80.0, a))


def test_ls_taps_gain_cap():
    """With cap=1 the fitted filter is non-expansive: |F(h)(w)| <= 1 for all w (DTFT of P:895-896,
    evaluated independently at random frequencies); without it the short fit over-amplifies."""
    xi = steps.xi_of(80.0, physics.ps2_per_km(-21.7), 21.4e9)
    rng = np.random.default_rng(3)
    w = rng.uniform(-np.pi, np.pi, 20000)
    for T in (3, 5, 9):
        k = np.arange(T) - (T - 1) // 2
        h = steps.ls_taps(xi, T, cap=1.0)
        assert np.abs(np.exp(-1j * np.outer(w, k)) @ h).max() <= 1.0 + 1e-6
        h0 = steps.ls_taps(xi, T)
        ratio = h0 / h
        assert np.allclose(ratio, ratio[0]) and abs(ratio[0].imag) < 1e-12 and ratio[0].real >= 1.0
