"""§8(f) NEXT-4: learned ESSM (filtered nonlinear steps) on the GPU vs the oracle
(oracle/essm.py) on the same fp32-rounded inputs: outputs rel-L2 <= 1e-5, every gradient
(dtaps per step, dgamma', deta per step) rel-L2 <= 1e-4, loss <= 1e-5."""
import numpy as np
import pytest
import torch

import ldbp_inputs as li
from oracle import essm

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


def model(seed, M, T, kap, sym):
    taps = li.random_sym_taps(seed, M, T, 0.1) if sym else li.random_general_taps(seed, M, T, 0.1)
    gamma = li.random_gamma(seed, M, -30.0, -5.0)
    g = np.random.default_rng(seed)
    eta = g.uniform(0.0, 1.0, (M, 2 * kap + 1))
    eta /= eta.sum(axis=1, keepdims=True)  # low-pass filters with unit DC gain (filtered DBP)
    return taps, gamma, eta


CASES = [
    # B, n, M, T, kappa, sym
    (2, 3000, 4, 5, 20, True),     # kappa = 20 (the paper's filter length), ragged tiles
    (3, 1024, 3, 9, 4, False),     # general taps
    (2, 50, 3, 3, 20, True),       # 2 kappa + 1 = 41 <= n = 50: halos wrap the block
    (1, 4096, 2, 15, 0, True),     # kappa = 0: the standard nonlinear step
]


@pytest.mark.parametrize("B,n,M,T,kap,sym", CASES)
def test_essm_forward_parity(P, B, n, M, T, kap, sym):
    x = li.gaussian_blocks(61, range(B), n, 1e-3)
    taps, gamma, eta = model(61, M, T, kap, sym)
    y = P.ldbp_essm_forward(dev(x), dev(taps), dev(gamma, np.float32), dev(eta, np.float32), symmetric=sym)
    yr = essm.forward(r32(x), r32(taps), r32(gamma), r32(eta))
    y = y.cpu().numpy()
    for b in range(B):
        assert rel(y[b], yr[b]) <= 1e-5, b


@pytest.mark.parametrize("B,n,M,T,kap,sym", CASES)
def test_essm_loss_grad_parity(P, B, n, M, T, kap, sym):
    x = li.gaussian_blocks(62, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(62, range(B), n, 1e-3, purpose="target")
    taps, gamma, eta = model(62, M, T, kap, sym)
    buf = P.ldbp_essm_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32), dev(eta, np.float32),
                                symmetric=sym).cpu().numpy()
    ref = essm.loss_grad(r32(x), r32(tgt), r32(taps), r32(gamma), r32(eta), symmetric=sym)
    NE = 2 * kap + 1
    assert abs(buf[0] - ref[0]) <= 1e-5 * ref[0]
    assert rel(buf[1:1 + M], ref[1:1 + M]) <= 1e-4
    dt, rdt = buf[1 + M:1 + M + 2 * M * T].reshape(M, -1), ref[1 + M:1 + M + 2 * M * T].reshape(M, -1)
    de, rde = buf[1 + M + 2 * M * T:].reshape(M, NE), ref[1 + M + 2 * M * T:].reshape(M, NE)
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= 1e-4, ("taps", i, rel(dt[i], rdt[i]))
        assert rel(de[i], rde[i]) <= 1e-4, ("eta", i, rel(de[i], rde[i]))
