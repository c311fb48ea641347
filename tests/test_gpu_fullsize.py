"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times: sampled
blocks against the oracle one by one, plus properties that hold at any size (sharding
linearity of the gradient buffer, equivariance)."""
import numpy as np
import pytest
import torch

import ldbp_inputs as li
from oracle import ldbp as O, physics, steps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2010_14258_b200 as P

    return P


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


POWERS_DBM = (-2.0, -1.0, 0.0, 1.0)  # training set P of §V-A


def gauss(B, n, seed):
    """Band-limited circular Gaussian blocks at per-block powers drawn from P (ldbp_inputs recipe)."""
    pw = li.dbm_to_w(li.pick_powers_dbm(seed, range(B), POWERS_DBM))
    return li.bandlimited_blocks_torch(seed, B, n, pw)


def ls_model(spans, sps, T):
    d, g = steps.dbp_plan(spans, 80.0, sps, 0.2, 1.3)
    taps = np.stack([steps.ls_taps(steps.xi_of(dd, physics.ps2_per_km(-21.7), 21.4e9), T, cap=1.0) for dd in d])
    return taps, g


def as_dev(taps, gamma):
    return (torch.from_numpy(taps.astype(np.complex64)).cuda(), torch.from_numpy(gamma.astype(np.float32)).cuda())


def c128(t):
    return t.cpu().numpy().astype(np.complex128)


@pytest.mark.parametrize("name,B,n,spans,sps,T", [
    ("C2", 256, 16384, 25, 1, 5),
    ("C4", 4096, 16384, 25, 4, 15),
])
def test_forward_full_size_sampled(P, name, B, n, spans, sps, T):
    taps, gamma = ls_model(spans, sps, T)
    ht, gt = as_dev(taps, gamma)
    x = gauss(B, n, 7)
    y = P.ldbp_forward(x, ht, gt)
    torch.cuda.synchronize()
    h64 = taps.astype(np.complex64).astype(np.complex128)
    g64 = gamma.astype(np.float32).astype(np.float64)
    for b in (0, B // 2 + 3, B - 1):
        ref = O.forward(c128(x[b:b + 1]), h64, g64)[0]
        assert rel(c128(y[b]), ref) <= 1e-5, (name, b)


@pytest.mark.parametrize("name,B,n,spans,sps,T,shards", [
    ("C3", 512, 16384, 25, 2, 9, 4),
    ("C5", 8192, 32768, 25, 1, 3, 2),
])
def test_loss_grad_full_size(P, monkeypatch, name, B, n, spans, sps, T, shards):
    taps, gamma = ls_model(spans, sps, T)
    ht, gt = as_dev(taps, gamma)
    x = gauss(B, n, 8)
    tgt = gauss(B, n, 9)
    full = P.ldbp_loss_grad(x, tgt, ht, gt).cpu().numpy()
    step = B // shards
    parts = sum(P.ldbp_loss_grad(x[s:s + step].contiguous(), tgt[s:s + step].contiguous(), ht, gt).cpu().numpy()
                for s in range(0, B, step))
    assert rel(parts, full) <= 1e-6
    # two sampled blocks vs the oracle, forced through the store-all schedule bench.py times (2 blocks
    # are below its 2^20-sample threshold; the whole timed batch is in test_gpu_timed_path.py)
    monkeypatch.setenv("LDBP_BWD_MODE", "1")
    monkeypatch.setenv("LDBP_STORE_ALL_MIN_SAMPLES", "0")
    M = len(gamma)
    h64 = taps.astype(np.complex64).astype(np.complex128)
    g64 = gamma.astype(np.float32).astype(np.float64)
    idx = [0, B - 1]
    sub = P.ldbp_loss_grad(x[idx].contiguous(), tgt[idx].contiguous(), ht, gt).cpu().numpy()
    ref = O.loss_grad(c128(x[idx]), c128(tgt[idx]), h64, g64, symmetric=True)
    assert abs(sub[0] - ref[0]) <= 1e-5 * ref[0]
    assert rel(sub[1:1 + M], ref[1:1 + M]) <= 1e-4
    dt, rdt = sub[1 + M:].reshape(M, -1), ref[1 + M:].reshape(M, -1)
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= 1e-4, (name, i)
