"""Regenerates the exact dot_chunked vectors of make_golden.dot_cases
(same rng stream) without importing the reference."""

import numpy as np

LENGTHS = [1, 2, 3, 31, 32, 33, 63, 64, 65, 100, 257, 1000, 1024, 4097]
CHUNKS = [1, 2, 7, 32, 33]


def dot_vectors():
    rng = np.random.default_rng(99)
    out = []
    for length in LENGTHS:
        for chunk in CHUNKS:
            x = rng.standard_normal(length)
            y = rng.standard_normal(length)
            out.append((length, chunk, x, y))
    return out
