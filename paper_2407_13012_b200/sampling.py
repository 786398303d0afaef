"""Shot sampling (reference: sampling.py:16-57).

`draw` runs the whole sampler on the device (csrc/sample.cu): probability tree
with the reference's pairwise association, one splitmix64 uniform per shot,
root-to-leaf descent and the cost gather.  Records keep draw order.  For large
shot counts the per-record tuples are built lazily; `indices`/`costs` expose the
arrays directly.
"""

from __future__ import annotations

import os

from collections import Counter

import numpy as np

from . import circuit
from .errors import ContractViolation


class SampleSet:
    """shots, seed and the (bitstring, cost) records in draw order."""

    __slots__ = ("shots", "seed", "_records", "indices", "costs")

    def __init__(self, shots: int, seed: int, records=None, *, indices=None, costs=None):
        self.shots = shots
        self.seed = seed
        self._records = tuple(records) if records is not None else None
        self.indices = indices
        self.costs = costs

    @property
    def records(self) -> tuple[tuple[int, float], ...]:
        if self._records is None:
            self._records = tuple(zip(self.indices.tolist(), self.costs.tolist()))
        return self._records

    def __eq__(self, other):
        if not isinstance(other, SampleSet):
            return NotImplemented
        return (self.shots, self.seed, self.records) == (other.shots, other.seed, other.records)

    __hash__ = None

    def __repr__(self) -> str:
        return f"SampleSet(shots={self.shots}, seed={self.seed})"


def draw(handle: circuit.SimHandle, shots: int, seed: int) -> SampleSet:
    """Sample the handle's current state (no re-simulation)."""
    if shots < 1:
        raise ContractViolation(f"shots must be >= 1, got {shots}")
    half = handle.state.half_view()
    if half is not None and os.environ.get("QSB_NO_HALF_SAMPLE", "0") in ("", "0"):
        # Z2-reduced state: draw from the lower half (no mirror copy; the same draws)
        idx, costs = handle.ctx.kernels.sample(half, handle.table.values.data, handle.n, int(shots), int(seed),
                                               half=True)
    else:
        idx, costs = handle.ctx.kernels.sample(handle.state.data, handle.table.values.data, handle.n, int(shots),
                                               int(seed))
    handle.ctx._count(handle.n + 2)
    return SampleSet(shots=shots, seed=seed, indices=idx, costs=costs)


def sample(handle: circuit.SimHandle, params: circuit.QaoaParams, shots: int, seed: int) -> SampleSet:
    """Simulate, then draw `shots` bitstrings with their objective values."""
    if shots < 1:
        raise ContractViolation(f"shots must be >= 1, got {shots}")
    circuit.simulate(handle, params)
    return draw(handle, shots, seed)


def best_of(samples: SampleSet) -> tuple[int, float]:
    """Minimal-cost record; ties go to the smaller bitstring."""
    if samples.indices is not None and samples._records is None:
        if samples.indices.shape[0] == 0:
            raise ContractViolation("best_of on an empty sample set")
        order = np.lexsort((samples.indices, samples.costs))
        i = int(order[0])
        return int(samples.indices[i]), float(samples.costs[i])
    if not samples.records:
        raise ContractViolation("best_of on an empty sample set")
    bit, cost = min(samples.records, key=lambda r: (r[1], r[0]))
    return bit, cost


def histogram(samples: SampleSet) -> dict[int, int]:
    """bitstring -> count, keys ascending."""
    if samples.indices is not None and samples._records is None:
        keys, counts = np.unique(samples.indices, return_counts=True)
        return {int(k): int(c) for k, c in zip(keys, counts)}
    return dict(sorted(Counter(b for b, _ in samples.records).items()))
