"""Progressive filter pruning with binary masks (paper §IV-C).

"the filters are successively shortened during the gradient-descent optimization by forcing
their outermost taps to zero ... the affected taps are then multiplied with a binary mask ...
each pruning step always removes the two outermost taps of a given filter", and "it is
generally beneficial to prune more taps in the beginning".

The mask is the ABI's `tap_mask` (uint8 [M][T]): ldbp_loss_grad multiplies the taps by it and
returns zero gradient for masked taps, ldbp_adam_update forces masked parameters and their Adam
moments to zero.  So pruning is host-side bookkeeping: this module builds the event schedule
and edits the device mask between iterations (an async device copy, no host sync).

Schedule (paper silent on details; SPEC's default, reading G18): all events inside the
first `frac` of the iterations, uniformly spaced, round-robin over the steps, longest current
filter first (ties: lowest step index).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def mask_for_lengths(lengths, taps: int) -> np.ndarray:
    """uint8 [M][T] mask keeping the central lengths[i] taps of each (odd) length-T filter."""
    kh = (taps - 1) // 2
    m = np.zeros((len(lengths), taps), dtype=np.uint8)
    for i, L in enumerate(lengths):
        if L < 1 or L % 2 == 0 or L > taps:
            raise ValueError(f"step {i}: target length {L} must be odd and in [1, {taps}]")
        k = (L - 1) // 2
        m[i, kh - k: kh + k + 1] = 1
    return m


def lengths_of(mask: np.ndarray) -> np.ndarray:
    return np.asarray(mask, dtype=np.int64).sum(axis=1)


@dataclass
class PruneSchedule:
    taps: int
    initial: list
    target: list
    iterations: int
    frac: float = 0.4
    events: list = field(default_factory=list)  # [(iteration, step)]

    @staticmethod
    def build(initial_lengths, target_lengths, iterations: int, taps: int | None = None, frac: float = 0.4):
        initial = [int(x) for x in initial_lengths]
        target = [int(x) for x in target_lengths]
        if len(initial) != len(target):
            raise ValueError("initial and target lengths differ in size")
        T = int(taps if taps is not None else max(initial))
        for a, b in zip(initial, target):
            if a % 2 == 0 or b % 2 == 0 or b > a or a > T:
                raise ValueError("lengths must be odd with target <= initial <= taps")
        n_events = sum((a - b) // 2 for a, b in zip(initial, target))
        cur = list(initial)
        order = []
        for _ in range(n_events):
            # longest filter that still has taps to remove; ties -> lowest index (round robin
            # emerges because the pruned filter becomes shorter than its peers)
            cand = [i for i in range(len(cur)) if cur[i] > target[i]]
            i = max(cand, key=lambda k: (cur[k], -k))
            order.append(i)
            cur[i] -= 2
        horizon = max(1, int(frac * iterations))
        its = [int(round((e + 1) * horizon / (n_events + 1))) for e in range(n_events)]
        return PruneSchedule(T, initial, target, iterations, frac, list(zip(its, order)))

    @property
    def n_events(self) -> int:
        return len(self.events)

    def initial_mask(self) -> np.ndarray:
        return mask_for_lengths(self.initial, self.taps)

    def mask_at(self, iteration: int) -> np.ndarray:
        """Mask after all events with event iteration <= `iteration`."""
        lengths = list(self.initial)
        for it, i in self.events:
            if it <= iteration:
                lengths[i] -= 2
        return mask_for_lengths(lengths, self.taps)

    def events_at(self, iteration: int):
        return [i for it, i in self.events if it == iteration]

    def apply(self, state, iteration: int) -> bool:
        """Update a TrainState's device mask for this iteration; returns True if it changed."""
        if not self.events_at(iteration):
            return False
        import torch

        state.set_mask(self.mask_at(iteration))
        return True
