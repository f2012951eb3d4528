"""Seeded synthetic inputs shared by the golden generator, the tests and
bench.py.  numpy's default_rng stream is platform
independent, so the GPU box regenerates the exact bytes the reference saw."""

import numpy as np


def make_case_input(n, r, seed, kind="gauss"):
    if kind == "diag21":
        return np.asfortranarray(np.diag([2.0, 1.0]))
    if kind == "shear11":
        return np.asfortranarray(np.array([[1.0, 1.0], [0.0, 1.0]]))
    if kind == "shear21":
        return np.asfortranarray(np.array([[2.0, 1.0], [0.0, 1.0]]))
    G = np.random.default_rng(seed).standard_normal((n, r))
    if kind == "gauss":
        return np.asfortranarray(G)
    if kind.startswith("graded"):
        # column grading 10^(-e*k/(r-1)), e = 12 or 10 (SURVEY.md §8(d) cfg 4)
        e = float(kind[len("graded"):])
        k = np.arange(r)
        return np.asfortranarray(G * 10.0 ** (-e * k / (r - 1)))
    raise ValueError(kind)
