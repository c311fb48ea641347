"""Pruning schedule (NEXT-3): paper rules and Example 2; GPU training keeps pruned taps at 0."""
import json
import os

import numpy as np
import pytest

from oracle import steps as osteps
from paper_2010_14258_b200.pruning import PruneSchedule, lengths_of, mask_for_lengths


def test_example2_event_count(golden_dir):
    """Example 2: 5 layers, T' = 11 -> T = 7: 10 pruning steps (every 10 of 100 its)."""
    g = json.load(open(os.path.join(golden_dir, "taps_counts.json")))
    sch = PruneSchedule.build(g["initial_lengths"], g["target_lengths"], iterations=100)
    assert sch.n_events == g["expected_events"] == osteps.pruning_events(g["initial_lengths"], g["target_lengths"])
    its = [it for it, _ in sch.events]
    assert its == sorted(its) and its[-1] <= 40  # front-loaded
    assert np.all(lengths_of(sch.mask_at(100)) == 7)


def test_outermost_pair_rule_and_monotone():
    """Each event removes the two outermost remaining taps of one filter."""
    T = 9
    sch = PruneSchedule.build([9] * 25, [5 if i % 2 == 0 else 3 for i in range(25)], iterations=1000)
    prev = sch.initial_mask()
    assert np.all(prev == 1)
    for it in sorted({it for it, _ in sch.events}):
        m = sch.mask_at(it)
        diff = prev.astype(int) - m.astype(int)
        assert np.all(diff >= 0)  # never un-prunes
        for i in np.nonzero(diff.sum(axis=1))[0]:
            removed = np.nonzero(diff[i])[0]
            kept = np.nonzero(m[i])[0]
            assert len(removed) == 2 and removed[0] + removed[1] == T - 1  # a symmetric pair
            assert removed[0] < kept.min() and removed[1] > kept.max()    # the outermost one
        np.testing.assert_array_equal(m, m[:, ::-1])  # symmetric
        prev = m
    # paper's headline model: alternating 5/3 taps -> 13*4 + 12*2 + 1 = 77 total taps
    assert osteps.total_impulse_length(lengths_of(prev)) == 77


def test_mask_lengths_validation():
    with pytest.raises(ValueError):
        mask_for_lengths([4], 9)
    with pytest.raises(ValueError):
        PruneSchedule.build([9], [11], 10)
    np.testing.assert_array_equal(mask_for_lengths([3], 7)[0], osteps.prune_mask(7, 3))


@pytest.mark.gpu
def test_training_with_pruning_keeps_pruned_taps_zero():
    import torch

    import ldbp_inputs as li
    import paper_2010_14258_b200 as P

    B, n, M, T = 4, 2048, 6, 9
    x = torch.from_numpy(li.gaussian_blocks(91, range(B), n, 1e-3).astype(np.complex64)).cuda()
    tgt = torch.from_numpy(li.gaussian_blocks(91, range(B), n, 1e-3, purpose="target").astype(np.complex64)).cuda()
    taps = li.random_sym_taps(91, M, T)
    gamma = li.random_gamma(91, M)
    st = P.TrainState.create(taps, gamma)
    sch = PruneSchedule.build([9] * M, [5, 3, 5, 3, 5, 3], iterations=20, frac=0.5)
    st.mask = torch.from_numpy(sch.initial_mask()).cuda()
    for it in range(20):
        sch.apply(st, it)
        P.ldbp_train_step(st, x, tgt)
    torch.cuda.synchronize()
    m = torch.from_numpy(sch.mask_at(20)).cuda().bool()
    t = st.taps
    assert torch.all(t[~m] == 0)
    assert torch.all(t[m] != 0)
    master = torch.view_as_complex(st.master[: 2 * M * T].view(M, T, 2))
    assert torch.all(master[~m] == 0)
    mm = st.m[: 2 * M * T].view(M, T, 2)
    assert torch.all(mm[~m] == 0)
