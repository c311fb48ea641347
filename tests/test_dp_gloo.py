"""World-size-2 gloo test of the data-parallel host logic on CPU.

Each rank computes its shard's gradient buffer with the CPU oracle (stand-in for the CUDA
loss_grad, which needs a GPU), the trainer all-reduces it over gloo and applies Adam.  Checks:
parameters stay identical across ranks and equal the single-process full-batch trajectory.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ldbp_inputs as li
from oracle import ldbp as O
from paper_2010_14258_b200.dp import DataParallelLDBP, shard

B, N, M, T, ITERS = 6, 64, 3, 5, 3


def _problem():
    x = li.gaussian_blocks(5, range(B), N, 1e-2)
    tgt = li.gaussian_blocks(5, range(B), N, 1e-2, purpose="target")
    taps = li.random_sym_taps(5, M, T)
    gamma = li.random_gamma(5, M)
    return x, tgt, taps, gamma


class OracleState:
    def __init__(self, taps, gamma):
        self.theta = O.pack_params(taps, gamma)
        self.m = np.zeros_like(self.theta)
        self.v = np.zeros_like(self.theta)
        self.t = 0

    def params(self):
        return O.unpack_params(self.theta, M, T)

    def adam(self, buf, n_global):
        self.t += 1
        self.theta, self.m, self.v = O.adam_update(np.asarray(buf), n_global, self.theta, self.m, self.v,
                                                   self.t, M, T)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, tgt, taps, gamma = _problem()
    mine = shard(rank, world, B)
    st = OracleState(taps, gamma)

    def lg(xl, tl):
        h, g = st.params()
        return torch.from_numpy(O.loss_grad(xl, tl, h, g, symmetric=True))

    tr = DataParallelLDBP(loss_grad_fn=lg, adam_fn=lambda buf, n: st.adam(buf.numpy(), n))
    assert tr.set_local_samples(len(mine) * N) == B * N
    losses = []
    for _ in range(ITERS):
        buf = tr.step(x[mine.start:mine.stop], tgt[mine.start:mine.stop])
        losses.append(float(buf[0]))
    gathered = [torch.zeros_like(torch.from_numpy(st.theta)) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(st.theta))
    if rank == 0:
        out.put((np.stack([g.numpy() for g in gathered]), losses))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_partition():
    for total in (1, 7, 8, 4096):
        for world in (1, 2, 3, 8):
            idx = [i for r in range(world) for i in shard(r, world, total)]
            assert idx == list(range(total))


def test_dp_gloo_world2_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    thetas, losses = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(thetas[0], thetas[1])
    # single-process reference trajectory on the full batch
    x, tgt, taps, gamma = _problem()
    st = OracleState(taps, gamma)
    ref_losses = []
    for _ in range(ITERS):
        h, g = st.params()
        buf = O.loss_grad(x, tgt, h, g, symmetric=True)
        ref_losses.append(buf[0])
        st.adam(buf, B * N)
    np.testing.assert_allclose(thetas[0], st.theta, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(losses, ref_losses, rtol=1e-12)
