"""The product's host-side init helpers agree with the independently written oracle ones."""
import numpy as np

from oracle import physics, steps
from paper_2010_14258_b200 import init as pinit


def test_schedule_matches_oracle():
    for sps in (1, 2, 4):
        d1, g1 = pinit.dbp_schedule(25, 80.0, sps)
        d2, g2 = steps.dbp_plan(25, 80.0, sps, 0.2, 1.3)
        np.testing.assert_allclose(d1, d2, rtol=1e-12)
        np.testing.assert_allclose(g1, g2, rtol=1e-12)


def test_inverse_cd_taps_match_oracle_ls():
    for T in (3, 5, 9, 15):
        for delta in (0.0, 20.0, 80.0):
            xi = steps.xi_of(delta, physics.ps2_per_km(-21.7), 21.4e9)
            h1 = pinit.inverse_cd_taps(delta, T, cap=None)
            h2 = steps.ls_taps(xi, T, n_grid=512)
            np.testing.assert_allclose(h1, h2, atol=1e-12)
            h1c = pinit.inverse_cd_taps(delta, T, cap=1.0)
            h2c = steps.ls_taps(xi, T, n_grid=512, cap=1.0)
            np.testing.assert_allclose(h1c, h2c, atol=1e-12)
