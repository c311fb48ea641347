"""GPU transmitted waveform (ldbp_tx_waveform) vs the oracle's modulate (Eq. (11), P:733-743;
SURVEY.md §8(c) G-2): sqrt(P) sps e^{j phi} F^-1 RRC F U s, circularly shifted by k samples.

Tolerance: the waveform is an output of fp32 FFTs -> rel-L2 <= 1e-5 per block (the §8(c) output
bound).  Covers one CTA per block (n <= 2^14), 2- and 4-CTA clusters (2^15, 2^16), sps 2 and 4,
shifts of either sign and beyond n, NULL shift / phase, and the bench's e2e target path (the
target built from symbol codes equals channel.link_blocks' target).
"""
import numpy as np
import pytest
import torch

import ldbp_inputs as li
from oracle import channel as OC

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2010_14258_b200 as P

    return P


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


QAM16 = (li.QAM16_LEVELS[:, None] + 1j * li.QAM16_LEVELS[None, :]).reshape(-1)  # code 4 i + q


@pytest.mark.parametrize("n,sps,B,with_aug", [(2048, 2, 3, True), (16384, 2, 2, True), (32768, 2, 2, True),
                                              (65536, 4, 1, True), (4096, 4, 2, False)])
def test_tx_waveform_vs_oracle(P, n, sps, B, with_aug):
    rng = np.random.default_rng(n + sps)
    K = n // sps
    codes = rng.integers(0, 16, size=(B, K)).astype(np.uint8)
    pw = (10.0 ** ((rng.uniform(-4, 6, B) - 30) / 10)).astype(np.float32)
    shift = rng.integers(-3 * n, 3 * n, size=B).astype(np.int32) if with_aug else None
    phase = rng.uniform(-np.pi, np.pi, B).astype(np.float32) if with_aug else None
    out = P.ldbp_tx_waveform(torch.from_numpy(codes).cuda(), torch.from_numpy(QAM16.astype(np.complex64)).cuda(),
                             torch.from_numpy(pw).cuda(), sps=sps,
                             shift=None if shift is None else torch.from_numpy(shift).cuda(),
                             phase=None if phase is None else torch.from_numpy(phase).cuda()).cpu().numpy()
    c32 = QAM16.astype(np.complex64).astype(np.complex128)
    for b in range(B):
        w = OC.modulate(c32[codes[b]], sps, float(pw[b]))
        if with_aug:
            w = np.roll(w, int(shift[b])) * np.exp(1j * np.float64(phase[b]))
        assert rel(out[b], w) <= 1e-5, (b, rel(out[b], w))


def test_tx_waveform_is_bench_target(P):
    """The e2e path of bench.py: targets built on the device from symbol codes + per-block
    power / shift / rotation equal the targets channel.link_blocks produces."""
    from paper_2010_14258_b200 import channel

    B, n = 8, 16384
    x, tgt = channel.link_blocks(3, range(B), n)
    codes, pw, shift, phase = channel.link_codes(3, range(B), n)
    out = P.ldbp_tx_waveform(codes, channel.qam16_table(), pw, sps=channel.RHO_D, shift=shift, phase=phase)
    t = tgt.cpu().numpy()
    o = out.cpu().numpy()
    for b in range(B):
        assert rel(o[b], t[b]) <= 1e-5, (b, rel(o[b], t[b]))


def test_tx_waveform_errors(P):
    from paper_2010_14258_b200._lib import LdbpError

    codes = torch.zeros((2, 1000), dtype=torch.uint8, device="cuda")  # n = 2000: not a power of two
    tab = torch.ones(16, dtype=torch.complex64, device="cuda")
    pw = torch.ones(2, dtype=torch.float32, device="cuda")
    with pytest.raises(LdbpError):
        P.ldbp_tx_waveform(codes, tab, pw, sps=2)
