"""Data-parallel LDBP training over the GPUs of one node.

One process per GPU (torchrun).  Blocks are independent circular frames, so rank r
of G owns the contiguous global block range ``shard(r, G, B_global)``; inputs are generated or
loaded per rank from the global block index, so the union is the same for any G.  The only
collective is one all-reduce (SUM) per iteration of the float64 gradient buffer
``[sum|e|^2 | dgamma[M] | dtaps[M][T][2]]`` (<= 7.6 KB at C3) through ``torch.distributed``
(NCCL over NVLink/NVSwitch on B200; gloo in the CPU tests).  Adam then runs identically on every
rank from the identical reduced buffer, so parameters stay bit-identical without a broadcast.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard(rank: int, world: int, total_blocks: int) -> range:
    """Contiguous global block indices owned by `rank` (balanced to within one block)."""
    base, extra = divmod(total_blocks, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class DataParallelLDBP:
    """Per-rank trainer.  ``loss_grad_fn(x, target) -> buf`` and ``adam_fn(buf, n_global)`` default
    to the CUDA ABI (``ldbp_loss_grad`` / ``ldbp_adam_update`` on ``state``); tests inject other
    implementations to exercise the host-side logic on CPU with the gloo backend."""

    state: object = None
    group: Optional[object] = None
    loss_grad_fn: Optional[Callable] = None
    adam_fn: Optional[Callable] = None
    n_global: float = 0.0
    # optional fused single-process step ``train_step_fn(x, target) -> buf`` (ldbp_train_step: one
    # launch for tiny problems); used when world == 1, where there is no exchange between the
    # gradient and Adam
    train_step_fn: Optional[Callable] = None
    # run the collectives even at world == 1 (a one-rank NCCL group on a single GPU exercises the
    # communicator and the fp64 all-reduce of the gradient buffer: tests/test_gpu_dp_nccl.py)
    force_collective: bool = False

    def __post_init__(self):
        if self.loss_grad_fn is None or self.adam_fn is None:
            from . import api

            st = self.state
            if self.loss_grad_fn is None:
                self.loss_grad_fn = lambda x, t: api.ldbp_loss_grad_state(st, x, t)
            if self.adam_fn is None:
                self.adam_fn = lambda buf, n: api.ldbp_adam_update(st, buf, n)

    @property
    def world(self) -> int:
        return dist.get_world_size(self.group) if dist.is_initialized() else 1

    def set_local_samples(self, local_samples: int) -> float:
        """n_global = sum over ranks of B_local * n (one small all-reduce at setup)."""
        t = torch.tensor([float(local_samples)], dtype=torch.float64,
                         device="cuda" if self._nccl() else "cpu")
        if self._exchange():
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        self.n_global = float(t.item())
        return self.n_global

    def _nccl(self) -> bool:
        return dist.is_initialized() and dist.get_backend(self.group) == "nccl"

    def _exchange(self) -> bool:
        return dist.is_initialized() and (self.world > 1 or self.force_collective)

    def step(self, x_local, target_local):
        """loss_grad (local) -> all_reduce(SUM) -> Adam.  Returns the reduced buffer."""
        if self.n_global <= 0:
            raise RuntimeError("call set_local_samples() first")
        if self.train_step_fn is not None and not self._exchange():
            return self.train_step_fn(x_local, target_local)
        buf = self.loss_grad_fn(x_local, target_local)
        if self._exchange():
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        self.adam_fn(buf, self.n_global)
        return buf
