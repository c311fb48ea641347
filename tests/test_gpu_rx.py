"""§8(f) NEXT-1: receiver-chain symbol loss on the GPU vs the oracle (same fp32-rounded inputs).

Matched filter = the decimating circular FIR of reading G19 (truncated periodic RRC impulse
response), genie phase, symbol error energy (Eq. (12)-(13)), and its gradient
through LDBP.  Tolerances as the hot path: loss <= 1e-5 rel, gradients rel-L2 <= 1e-4.
"""
import numpy as np
import pytest
import torch

import ldbp_inputs as li
from oracle import channel, ldbp as O, receiver

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2010_14258_b200 as P

    return P


def dev(a, dtype=np.complex64):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).astype(dtype))).cuda()


def r32(a):
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return a.astype(np.complex64).astype(np.complex128)
    return a.astype(np.float32).astype(np.float64)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def link(seed, B, K, sps, snr_noise=0.05):
    """Symbols, powers and a received-like waveform: modulated 16-QAM plus a perturbation."""
    s = np.stack([li.qam16(li.rng(seed, b, "symbols"), K) for b in range(B)])
    pw = li.dbm_to_w(li.pick_powers_dbm(seed, range(B), (-2.0, -1.0, 0.0, 1.0)))
    y = np.stack([channel.modulate(s[b], sps, pw[b]) for b in range(B)])
    y = y * np.exp(0.7j) + snr_noise * np.sqrt(pw)[:, None] * li.cn(li.rng(seed, 0, "augment"), y.shape)
    return s, pw, y


@pytest.mark.parametrize("B,K,sps,span", [
    (3, 1024, 2, 32),    # one chunk per block
    (2, 5000, 2, 32),    # several chunks, ragged last chunk
    (2, 700, 1, 16),     # sps = 1
    (2, 1500, 4, 8),     # sps = 4
    (1, 96, 2, 40),      # MF longer than half the block (wraps)
])
def test_rx_loss_grad_parity(P, B, K, sps, span):
    s, pw, y = link(11, B, K, sps)
    h = receiver.rrc_fir_taps(sps, 0.1, span)
    errs, gy = P.ldbp_rx_loss_grad(dev(y), dev(s), dev(pw, np.float32), dev(h, np.float32), sps=sps)
    errs, gy = errs.cpu().numpy(), gy.cpu().numpy()
    re, rgy, _ = receiver.rx_loss_grad(r32(y), r32(s), r32(pw), r32(h), sps)
    for b in range(B):
        assert abs(errs[b] - re[b]) <= 1e-5 * re[b], (b, errs[b], re[b])
        assert rel(gy[b], rgy[b]) <= 1e-4, (b, rel(gy[b], rgy[b]))
    # loss-only call gives the same errors
    e2, g2 = P.ldbp_rx_loss_grad(dev(y), dev(s), dev(pw, np.float32), dev(h, np.float32), sps=sps, need_grad=False)
    assert g2 is None and torch.equal(e2.cpu(), torch.from_numpy(errs))


@pytest.mark.parametrize("mode", ["0", "1"])
def test_rx_train_grad_parity(P, monkeypatch, mode):
    """Receiver-chain loss through LDBP: buf = [sum errs | dgamma | dtaps] vs the oracle chain
    (forward, rx_loss_grad, adjoint) on the same inputs; both activation schedules."""
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    B, K, sps, M, T = 3, 2048, 2, 6, 5
    s, pw, x = link(12, B, K, sps, snr_noise=0.02)
    taps = li.random_sym_taps(12, M, T, 0.05)
    gamma = li.random_gamma(12, M, -3.0, -1.0)
    h = receiver.rrc_fir_taps(sps, 0.1, 32)
    buf = P.ldbp_rx_train_grad(dev(x), dev(s), dev(pw, np.float32), dev(h, np.float32), dev(taps),
                               dev(gamma, np.float32), sps=sps).cpu().numpy()
    yo = O.forward(r32(x), r32(taps), r32(gamma))
    errs, gyo, _ = receiver.rx_loss_grad(yo, r32(s), r32(pw), r32(h), sps)
    rdt, rdg, _ = O.backward(r32(x), gyo, r32(taps), r32(gamma))
    rdt = O.sym_fold(rdt)
    assert abs(buf[0] - errs.sum()) <= 1e-5 * errs.sum()
    assert rel(buf[1:1 + M], rdg) <= 1e-4
    dt = buf[1 + M:].reshape(M, T, 2)
    dt = dt[..., 0] + 1j * dt[..., 1]
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= 1e-4, i


# ---- exact circulant matched filter (Eq. (12) as written: M is the circulant, no truncation) ----
@pytest.mark.parametrize("B,K,sps,weighted", [
    (3, 512, 2, False),     # one CTA per block
    (2, 8192, 2, True),     # n = 2^14 (C3 block), per-block weights
    (2, 16384, 2, False),   # n = 2^15 (C5 block): 2-CTA cluster
    (2, 1024, 4, True),     # sps = 4
    (2, 4096, 1, False),    # sps = 1
])
def test_rx_exact_loss_grad_parity(P, B, K, sps, weighted):
    s, pw, y = link(13, B, K, sps)
    w = np.linspace(0.5, 2.0, B) if weighted else None
    errs, gy = P.ldbp_rx_exact_loss_grad(dev(y), dev(s), dev(pw, np.float32), sps=sps,
                                         weights=None if w is None else dev(w, np.float32))
    errs, gy = errs.cpu().numpy(), gy.cpu().numpy()
    re, rgy = receiver.rx_loss_grad_exact(r32(y), r32(s), r32(pw), sps,
                                          weights=None if w is None else r32(w))
    for b in range(B):
        assert abs(errs[b] - re[b]) <= 1e-5 * re[b], (b, errs[b], re[b])
        assert rel(gy[b], rgy[b]) <= 1e-4, (b, rel(gy[b], rgy[b]))
    e2, g2 = P.ldbp_rx_exact_loss_grad(dev(y), dev(s), dev(pw, np.float32), sps=sps, need_grad=False)
    assert g2 is None and np.allclose(e2.cpu().numpy(), errs, rtol=0, atol=0)


@pytest.mark.parametrize("mode", ["0", "1"])
def test_rx_exact_train_grad_parity(P, monkeypatch, mode):
    """Exact receiver-chain loss through LDBP vs the oracle chain (forward, exact MF loss and its
    gradient, adjoint), both activation schedules, with per-block weights."""
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_STORE_ALL_MIN_SAMPLES", "0")
    B, K, sps, M, T = 3, 2048, 2, 6, 5
    s, pw, x = link(14, B, K, sps, snr_noise=0.02)
    w = np.array([1.0, 0.5, 2.0])
    taps = li.random_sym_taps(14, M, T, 0.05)
    gamma = li.random_gamma(14, M, -3.0, -1.0)
    buf = P.ldbp_rx_exact_train_grad(dev(x), dev(s), dev(pw, np.float32), dev(taps), dev(gamma, np.float32),
                                     sps=sps, weights=dev(w, np.float32)).cpu().numpy()
    yo = O.forward(r32(x), r32(taps), r32(gamma))
    errs, gyo = receiver.rx_loss_grad_exact(yo, r32(s), r32(pw), sps, weights=r32(w))
    rdt, rdg, _ = O.backward(r32(x), gyo, r32(taps), r32(gamma))
    rdt = O.sym_fold(rdt)
    L = float(np.sum(r32(w) * errs))
    assert abs(buf[0] - L) <= 1e-5 * L
    # dgamma'_i per step.  The last step's sum_t Im(gy_t conj(y_t)) |y_t|^2 cancels strongly (the
    # loss is stationary in the global phase at the genie phi), so it is checked against
    # the magnitude of its terms; every other step against its own value.
    cancel = np.sum(np.abs(np.imag(gyo * np.conj(yo)) * np.abs(yo) ** 2))
    for i in range(M):
        scale = abs(rdg[i]) if i < M - 1 else max(abs(rdg[i]), cancel)
        assert abs(buf[1 + i] - rdg[i]) <= 1e-4 * scale, (i, buf[1 + i], rdg[i], scale)
    dt = buf[1 + M:].reshape(M, T, 2)
    dt = dt[..., 0] + 1j * dt[..., 1]
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= 1e-4, i
