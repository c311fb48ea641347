"""Inputs keyed by global block index (VERDICT r1 Next #5): the blocks a rank
draws depend only on their global indices, so the union over ranks of a sharded batch is the
same array for any number of ranks G (checked on the CPU device; bench.py draws on the GPU)."""
import numpy as np
import torch

import ldbp_inputs as li
from paper_2010_14258_b200.dp import shard


def test_union_of_shards_is_independent_of_world_size():
    B, n = 10, 256
    pw = li.dbm_to_w(li.pick_powers_dbm(3, range(B), (-2.0, -1.0, 0.0, 1.0)))
    full = li.bandlimited_blocks_keyed_torch(3, range(B), n, pw, device="cpu").numpy()
    for G in (2, 3, 4):
        parts = []
        for r in range(G):
            blk = list(shard(r, G, B))
            parts.append(li.bandlimited_blocks_keyed_torch(3, blk, n, pw[blk], device="cpu").numpy())
        assert np.array_equal(np.concatenate(parts), full), G


def test_keyed_blocks_statistics():
    """Band-limited (no energy outside the occupied RRC band) with the requested mean power."""
    n = 4096
    x = li.bandlimited_blocks_keyed_torch(5, range(4), n, 2e-3, device="cpu").numpy().astype(np.complex128)
    spec = np.abs(np.fft.fft(x, axis=-1)) ** 2
    out = li.bandlimited_mask(n) == 0
    assert spec[:, out].sum() <= 1e-10 * spec.sum()
    p = np.mean(np.abs(x) ** 2, axis=-1)
    assert np.all(np.abs(p / 2e-3 - 1) < 0.1)
    # distinct keys give distinct blocks; targets differ from signals
    t = li.bandlimited_blocks_keyed_torch(5, range(4), n, 2e-3, device="cpu", purpose="target").numpy()
    assert not np.allclose(x[0], x[1]) and not np.allclose(x, t)
    assert torch.is_tensor(li.bandlimited_blocks_keyed_torch(5, [0], 8, 1.0, device="cpu"))
