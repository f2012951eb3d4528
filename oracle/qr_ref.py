"""numpy restatement of hjsvd.factory.qr_shorten (factory.py:300-334).

TEST INFRASTRUCTURE, NOT PRODUCT: only tests/ import it, as the checker of
the GPU QR shortening.  numpy's norm / dot use BLAS reduction orders, so the
GPU result is compared to this one to rounding, not bit for bit."""

import numpy as np


def qr_shorten_numpy(G):
    A = np.array(G, dtype=np.float64, order="F")
    n, r = A.shape
    vs = []
    for k in range(r):
        x = A[k:, k]
        normx = float(np.linalg.norm(x))
        sgn = 1.0 if x[0] >= 0.0 else -1.0
        alpha = -sgn * normx
        v = x.copy()
        v[0] -= alpha
        beta = 2.0 / float(v @ v)
        A[k:, k:] -= np.outer(beta * v, v @ A[k:, k:])
        A[k, k] = alpha
        A[k + 1:, k] = 0.0
        vs.append((k, v, beta))
    R = np.triu(A[:r, :])
    Q = np.eye(n, r, order="F")
    for k, v, beta in reversed(vs):
        Q[k:, :] -= np.outer(beta * v, v @ Q[k:, :])
    flip = np.diag(R) < 0.0
    R[flip, :] *= -1.0
    Q[:, flip] *= -1.0
    return np.asfortranarray(R), np.asfortranarray(Q)
