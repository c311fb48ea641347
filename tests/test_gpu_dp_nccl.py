"""Row a9 on hardware (P:296-299 mini-batches across GPUs): the
data-parallel trainer's exchange step through a real NCCL communicator.

A GPU box of this run has one GPU, so the group has ONE rank: `force_collective` makes the
trainer run its collectives anyway — NCCL communicator creation on cuda:0, the float64 all-reduce
(SUM) of the device-resident gradient buffer [sum|e|^2 | dgamma' | dtaps] in stream order between
`ldbp_loss_grad` and `ldbp_adam_update`, and the n_global reduction.  With one rank the
reduction is the identity, so the result must equal the collective-free path bit for bit, and the
reduced buffer must match the fp64 oracle within the gradient tolerance.  The two-rank logic
(sharding, sum over ranks, identical Adam on every rank) is covered on CPU with gloo
(tests/test_dp_gloo.py).
"""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import ldbp_inputs as li
from oracle import ldbp as O

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


@pytest.fixture()
def nccl_world1():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        yield
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,n,M,T", [(6, 4096, 6, 9), (4, 1024, 4, 3)])
def test_dp_step_through_nccl_allreduce(P, nccl_world1, monkeypatch, B, n, M, T):
    from paper_2010_14258_b200.dp import DataParallelLDBP

    monkeypatch.setenv("LDBP_TINY", "0")  # loss_grad -> exchange -> Adam as separate launches
    x = li.gaussian_blocks(91, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(91, range(B), n, 1e-3, purpose="target")
    taps = li.random_sym_taps(91, M, T, 0.1)
    gamma = li.random_gamma(91, M)
    dx, dt = dev(x), dev(tgt)

    plain = P.TrainState.create(taps, gamma)
    comm = P.TrainState.create(taps, gamma)
    tr = DataParallelLDBP(state=comm, force_collective=True)
    assert dist.get_backend() == "nccl" and tr._nccl() and tr.world == 1
    assert tr.set_local_samples(B * n) == float(B * n)  # the setup all-reduce, on the device

    ref = O.loss_grad(r32(x), r32(tgt), r32(taps), r32(gamma), symmetric=True)
    for it in range(3):
        b_plain = P.ldbp_loss_grad(dx, dt, plain.taps, plain.gamma)
        P.ldbp_adam_update(plain, b_plain, B * n)
        b_comm = tr.step(dx, dt)  # loss_grad -> NCCL all_reduce(SUM, fp64) -> Adam
        torch.cuda.synchronize()
        assert b_comm.is_cuda and b_comm.dtype == torch.float64
        assert torch.equal(b_comm, b_plain)  # one rank: SUM is the identity, bit for bit
        if it == 0:
            got = b_comm.cpu().numpy()
            assert abs(got[0] - ref[0]) <= 1e-5 * ref[0]
            assert rel(got[1:1 + M], ref[1:1 + M]) <= 1e-4
            assert rel(got[1 + M:], ref[1 + M:]) <= 1e-4
    assert torch.equal(comm.master, plain.master)
    assert torch.equal(comm.taps, plain.taps) and torch.equal(comm.gamma, plain.gamma)
