"""Pins of the counter-based ASE generator shared by the oracle's callers and the GPU channel kernel
(ldbp_inputs.philox4x32_10 / ase_cn_philox; the CUDA side is ldbp_ssfm.cuh ase_philox_cn)."""
import numpy as np

import ldbp_inputs as li


def test_philox4x32_10_known_answers():
    """Known-answer vectors of Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers:
    as easy as 1, 2, 3", SC'11; the Random123 distribution's kat_vectors)."""
    kat = [
        ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
        ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
        ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
         (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
    ]
    for ctr, key, want in kat:
        got = li.philox4x32_10(*[np.array([c]) for c in ctr], *key)
        assert tuple(int(v[0]) for v in got) == want


def test_ase_draws_are_cn01_and_keyed():
    z = li.ase_cn_philox(201014258, 3, 1, 1 << 16)
    assert abs(np.mean(np.abs(z) ** 2) - 1.0) < 0.02          # E|z|^2 = 1
    assert abs(np.mean(z)) < 0.02
    assert abs(np.mean(z.real ** 2) - 0.5) < 0.02 and abs(np.mean(z.real * z.imag)) < 0.02  # circular
    # Gaussian 4th moment: E|z|^4 = 2 for CN(0, 1)
    assert abs(np.mean(np.abs(z) ** 4) - 2.0) < 0.1
    # keyed: other span / block / seed give other draws; same key is reproducible
    assert not np.allclose(z, li.ase_cn_philox(201014258, 3, 2, 1 << 16))
    assert not np.allclose(z, li.ase_cn_philox(201014258, 4, 1, 1 << 16))
    assert np.array_equal(z, li.ase_cn_philox(201014258, 3, 1, 1 << 16))
    # prefixes agree (sample i depends only on i)
    assert np.array_equal(li.ase_cn_philox(7, 0, 0, 100), li.ase_cn_philox(7, 0, 0, 1000)[:100])
