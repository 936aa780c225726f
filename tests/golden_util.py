"""Helpers shared by tests/golden/make_golden.py and the GPU parity tests for
fixtures of grids too large to commit whole (configs 2 and 3): a fixed,
seed-free sample of (component, node) entries and size-independent
whole-field checksums."""
import numpy as np

SAMPLE_MULT = 2654435761  # odd, not a multiple of 3: a bijection mod 9 * 2^k
SAMPLE_OFF = 12345


def sample_index(count, total):
    """`count` distinct flat indices into a field of `total` entries,
    idx_k = (k * SAMPLE_MULT + SAMPLE_OFF) mod total (no RNG: identical on
    every numpy version)."""
    k = np.arange(count, dtype=np.uint64)
    assert np.gcd(SAMPLE_MULT, total) == 1 and count <= total
    return ((k * np.uint64(SAMPLE_MULT) + np.uint64(SAMPLE_OFF)) % np.uint64(total)).astype(np.int64)


def checksums(x, ncomp):
    """Per-component sum and sum of squares (float64, numpy pairwise order):
    whole-field properties the sampled entries cannot show."""
    x = np.asarray(x).reshape(ncomp, -1)
    return np.stack([x.sum(axis=1), np.einsum("ij,ij->i", x, x)])


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
