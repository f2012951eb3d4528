"""ctypes front end of the CPU oracle (oracle/hsvd_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT: only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs import this module.  It restates the
reference's pointwise HSVD (/root/reference/pkg/src/hjsvd/solver.py:179-269
and _kernels.py:32-251) with the same IEEE operation order, and is pinned
bit-for-bit to the reference by tests/golden (tests/test_oracle_golden.py).
"""

import ctypes
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc_hsvd.so")
_lib = None

EPS = 2.0 ** -52
TEPS = 2.0 ** -27

_d = ctypes.c_double
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build():
    """Compile liborc_hsvd.so with the committed Makefile (gcc, no contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_dot_chunked.restype = _d
        L.orc_dot_chunked.argtypes = [_p, _p, _i64, _i64]
        L.orc_fused_pair_update.restype = None
        L.orc_fused_pair_update.argtypes = [_p, _p, _i64, _d, _d, _d]
        L.orc_rotation_tc.restype = ctypes.c_int
        L.orc_rotation_tc.argtypes = [_d, _d, _d, _i64, ctypes.POINTER(_d),
                                      ctypes.POINTER(_d)]
        L.orc_step_blocks.restype = ctypes.c_int
        L.orc_step_blocks.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p, _p,
                                      _p, _p, _p, _p, _i64, _i64, _d, _d,
                                      ctypes.c_int, _i64, _p, _p]
        L.orc_stepper_init.restype = None
        L.orc_stepper_init.argtypes = [_i64, _p, _p, _p, _p]
        L.orc_advance_stepper.restype = None
        L.orc_advance_stepper.argtypes = [_p, _p, _p, _p, _i64, _i64]
        L.orc_sort_diagonal.restype = None
        L.orc_sort_diagonal.argtypes = [_p, _p, _p, _i64, _i64]
        L.orc_check_convergence.restype = ctypes.c_int
        L.orc_check_convergence.argtypes = [_p, _i64]
        L.orc_precompute.restype = _i64
        L.orc_precompute.argtypes = [_p, _i64, _i64, _i64, _i64, _p]
        L.orc_drive.restype = ctypes.c_int
        L.orc_drive.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _d, _d,
                                ctypes.c_int, ctypes.c_int, _i64, _i64,
                                ctypes.c_int, ctypes.c_int, _p, _p, _p, _p,
                                _p, _p, _p]
        L.orc_sample_steps.restype = _i64
        L.orc_sample_steps.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _i64,
                                       ctypes.c_int, ctypes.POINTER(_d)]
        L.orc_bp_factor.restype = ctypes.c_int
        L.orc_bp_factor.argtypes = [_p, _i64, _d, _p, _p, _p, _p, _p]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def dot_chunked(x, y, chunk=32):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return lib().orc_dot_chunked(_ptr(x), _ptr(y), x.shape[0], chunk)


def fused_pair_update(x, y, t, c, s):
    """In place on contiguous float64 vectors (reference _kernels.py:62-75)."""
    lib().orc_fused_pair_update(_ptr(x), _ptr(y), x.shape[0], t, c, s)


def rotation_tc(a_ii, a_jj, a_ij, hyp):
    t, c = _d(), _d()
    st = lib().orc_rotation_tc(a_ii, a_jj, a_ij, hyp, ctypes.byref(t),
                               ctypes.byref(c))
    return t.value, c.value, st


def stepper_init(r):
    ip, jp, ib, jb = (np.empty(r // 2, np.int64) for _ in range(4))
    lib().orc_stepper_init(r, _ptr(ip), _ptr(jp), _ptr(ib), _ptr(jb))
    return ip, jp, ib, jb


def advance_stepper(ip, jp, ib, jb, r):
    lib().orc_advance_stepper(_ptr(ip), _ptr(jp), _ptr(ib), _ptr(jb),
                              ip.shape[0], r)


def sort_diagonal(d, rho, jsign, p):
    lib().orc_sort_diagonal(_ptr(d), _ptr(rho), _ptr(jsign), d.shape[0], p)


def precompute(G, chunk=32):
    G = np.asfortranarray(G, dtype=np.float64)
    n, r = G.shape
    d = np.empty(r)
    bad = lib().orc_precompute(_ptr(G), n, r, n, chunk, _ptr(d))
    return d, int(bad)


def step_blocks(G, V, d, rho, jsign, iblk, jblk, C, k0, k1, eps=EPS,
                teps=TEPS, use_skip=True, chunk=32):
    """Reference step_blocks (_kernels.py:188-235) on F-ordered arrays."""
    n = G.shape[0]
    stats = np.zeros(3)
    err = np.full(3, -1, np.int64)
    st = lib().orc_step_blocks(
        _ptr(G), n, n, _ptr(V), 0 if V is None else V.shape[0],
        0 if V is None else V.shape[0], _ptr(d), _ptr(rho), _ptr(jsign),
        _ptr(iblk), _ptr(jblk), _ptr(C), k0, k1, eps, teps, int(use_skip),
        chunk, _ptr(stats), _ptr(err))
    return st, stats, err


def drive(G, signs, p, max_sweeps=30, eps=EPS, teps=None, accumulate_v=True,
          use_rel_orth_skip=True, chunk=32, workers=1, schedule="modulus",
          sort=True):
    """Whole reference drive (solver.py:179-269).  Returns a namespace with
    the HsvdResult fields, or raises RuntimeError(status, err)."""
    if teps is None:
        teps = float(np.sqrt(eps) / 2.0)
    G = np.asfortranarray(G, dtype=np.float64)
    n, r = G.shape
    signs = np.ascontiguousarray(signs, dtype=np.int8)
    sigma = np.empty(r)
    lam = np.empty(r)
    U = np.empty((n, r), order="F")
    V = np.empty((r, r), order="F") if accumulate_v else None
    info = np.zeros(4, np.int64)
    tele = np.zeros((max(max_sweeps, 1), 4))
    err = np.full(3, -1, np.int64)
    st = lib().orc_drive(
        _ptr(G), n, r, _ptr(signs), p, max_sweeps, eps, teps,
        int(accumulate_v), int(use_rel_orth_skip), chunk, workers,
        int(schedule == "row-cyclic"), int(sort), _ptr(sigma), _ptr(lam),
        _ptr(U), _ptr(V), _ptr(info), _ptr(tele), _ptr(err))
    if st != 0:
        raise RuntimeError(st, tuple(int(e) for e in err))
    sweeps = int(info[0])
    stop = {0: "orthogonal", 1: "quadratic", 2: "max_sweeps"}[int(info[1])]
    telemetry = [(int(t[0]), int(t[1]), int(t[2]), float(t[3]))
                 for t in tele[:sweeps]]
    return SimpleNamespace(sigma=sigma, U=U, lam=lam, Vinv_t=V,
                           sweeps_used=sweeps, stop_reason=stop,
                           rotations=int(info[2]), skips=int(info[3]),
                           telemetry=telemetry)


def sample_steps(G, signs, p, steps, workers, accumulate_v=True):
    """Bounded CPU-baseline sample: `steps` modulus steps of sweep 0 after
    precompute + sort.  Returns (rotations, seconds spent in the steps)."""
    G = np.asfortranarray(G, dtype=np.float64)
    n, r = G.shape
    signs = np.ascontiguousarray(signs, dtype=np.int8)
    el = _d()
    rot = int(lib().orc_sample_steps(_ptr(G), n, r, _ptr(signs), p, steps,
                                     workers, int(accumulate_v), ctypes.byref(el)))
    return rot, el.value


def bp_factor(M):
    """Bunch-Parlett factor of a symmetric M, bit-identical to
    hjsvd.factory.bunch_parlett_factor (factory.py:270-282): returns
    (G column-major, signs (+1 first), perm, p); raises ArithmeticError on a
    numerical singularity."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    n = M.shape[0]
    thresh = n * EPS * np.linalg.norm(M, "fro")
    G = np.zeros((n, n), order="F")
    signs = np.zeros(n, np.int8)
    perm = np.zeros(n, np.int64)
    p = np.zeros(1, np.int64)
    stage = np.zeros(1, np.int64)
    st = lib().orc_bp_factor(_ptr(M), n, thresh, _ptr(G), _ptr(signs), _ptr(perm), _ptr(p),
                             _ptr(stage))
    if st == 3:
        raise ArithmeticError(f"numerical singularity at stage {int(stage[0])}")
    return G, signs, perm, int(p[0])
