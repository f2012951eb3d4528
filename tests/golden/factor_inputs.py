"""Seeded symmetric inputs of the factorization goldens (regenerable anywhere
with numpy; the reference-generated spectra travel as factor_inputs.npz)."""

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def make_input(kind, n, seed):
    """kind: sym (X + X^T), smalldiag (X + X^T with the diagonal scaled by
    1e-3: 2x2 pivots), ints (small integers: many exact ties in the pivot
    search), diag (fixed diagonal), offdiag ([[0, 1], [1, 0]]), ones
    (singular), spectrum (reference generate_symmetric, stored in the npz)."""
    if kind == "spectrum":
        return np.load(os.path.join(HERE, "factor_inputs.npz"))[f"M_{n}_{seed}"]
    if kind == "diag":
        return np.diag([4.0, -1.0])
    if kind == "offdiag":
        return np.array([[0.0, 1.0], [1.0, 0.0]])
    if kind == "ones":
        return np.ones((n, n))
    rng = np.random.default_rng(seed)
    if kind == "ints":
        X = rng.integers(-3, 4, (n, n)).astype(np.float64)
        return X + X.T
    X = rng.standard_normal((n, n))
    M = X + X.T
    if kind == "smalldiag":
        M[np.diag_indices(n)] *= 1e-3
    return M
