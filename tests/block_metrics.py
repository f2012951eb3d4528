"""Shared accuracy metrics for block-mode parity (test infrastructure)."""

import numpy as np


def sigma_class_reldiff(sig_a, lam_a, sig_b, lam_b):
    """max relative difference of sigma per sign class after sorting (the
    reference's own comparison convention, test_solver.py:129, 135)."""
    out = 0.0
    for sgn in (1, -1):
        a = np.sort(np.asarray(sig_a)[np.sign(lam_a) == sgn])
        b = np.sort(np.asarray(sig_b)[np.sign(lam_b) == sgn])
        assert a.shape == b.shape
        if a.size:
            out = max(out, float(np.max(np.abs(a - b) / np.abs(b))))
    return out


def residuals(G, res, signs):
    """dU = ||U^T U - I||_F, vjv = ||V^T J V - J||_F / ||V||_F^2,
    recon = ||G - U S V^T||_F / ||G||_F with V = J V^{-T} J."""
    U = np.asarray(res.U)
    r = U.shape[1]
    s = signs.astype(np.float64)
    out = {"dU": float(np.linalg.norm(U.T @ U - np.eye(r)))}
    if res.Vinv_t is not None:
        V = s[:, None] * np.asarray(res.Vinv_t) * s[None, :]
        out["vjv"] = float(np.linalg.norm(V.T @ (s[:, None] * V) - np.diag(s))
                           / np.linalg.norm(V) ** 2)
        out["recon"] = float(np.linalg.norm(G - (U * np.asarray(res.sigma)) @ V.T)
                             / np.linalg.norm(G))
    return out
