"""Reproducible random streams keyed by (seed, *path) -- rng.py:17-33 of the
reference.  Sample indices must be bit-identical to the reference's, so the
draw uses the same numpy Philox/SeedSequence construction on the host (index
generation is host work in the reference too; it is overlapped with device
passes by the solver)."""

import numpy as np

GRAD_STREAM = 0
HESS_STREAM = 1
SPLIT_STREAM = 2
SHUFFLE_STREAM = 3
POWER_STREAM = 4

_MASK64 = (1 << 64) - 1


def stream_rng(seed, *path):
    """numpy Generator on Philox(SeedSequence([seed, *path])) (64-bit masked words)."""
    words = [int(seed) & _MASK64]
    words.extend(int(p) & _MASK64 for p in path)
    return np.random.Generator(np.random.Philox(seed=np.random.SeedSequence(words)))
