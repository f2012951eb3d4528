"""Eigen-pipeline front end: symmetric M -> factor pair (G, J) on the GPU.

Mirrors hjsvd.factory (/root/reference/pkg/src/hjsvd/factory.py): the same
names, dataclasses, constants and exceptions.  ``bunch_parlett_factor`` runs
the reference's complete-pivoting Bunch-Parlett factorization in
double-double on the device (csrc/hsvd_factor.cu, C entry hsvd_bp_factor)
and returns the reference's factor bit for bit.  ``qr_shorten`` is the
reference's Householder QR of a tall factor on the device (hsvd_qr_shorten;
plain fp64, equal to the reference's to rounding).  The eigenvalues of M
come from the HSVD of (G, J): lambda = sigma^2 * j (``eigvalsh``).
"""

import math
from dataclasses import dataclass

import ctypes

import numpy as np

from . import _lib
from ._device import ptr, require_cuda, stream_handle
from .errors import ShapeError
from .linalg import EPS, SignatureVector

#: complete-pivoting 2x2 threshold constant (factory.py:21)
ALPHA = (1.0 + math.sqrt(17.0)) / 8.0

#: relative spectral gap around zero (factory.py:24)
GAP = 1e-5


@dataclass(frozen=True)
class SpectrumSpec:
    """Random spectrum: n values uniform in [-a, -a*GAP] u [a*GAP, a]
    (factory.py:28-47); pos_count pins the number of positive values."""

    n: int
    a: float
    seed: int
    pos_count: int = None

    def __post_init__(self):
        if self.n < 2:
            raise ShapeError("n must be >= 2")
        if not self.a > 0.0:
            raise ValueError("a must be positive")
        if self.pos_count is not None and not 0 <= self.pos_count <= self.n:
            raise ValueError("pos_count must lie in [0, n]")


@dataclass(frozen=True)
class FactorPair:
    """Factor G with signature J (positives leading) and the symmetric
    permutation applied by the factorization (factory.py:50-57)."""

    G: np.ndarray
    J: SignatureVector
    perm: np.ndarray = None


@dataclass(frozen=True)
class TestBundle:
    """One generated instance: matrix, exact spectrum, and its factor
    (factory.py:60-66)."""

    __test__ = False  # not a pytest class

    M: np.ndarray
    lambda_true: np.ndarray  # sorted ascending
    factor: FactorPair
    spec: SpectrumSpec = None


def draw_spectrum(spec, rng):
    """Eigenvalues honoring the spectral gap (factory.py:69-76)."""
    mags = rng.uniform(spec.a * GAP, spec.a, spec.n)
    if spec.pos_count is None:
        signs = rng.integers(0, 2, spec.n) * 2 - 1
    else:
        signs = np.where(np.arange(spec.n) < spec.pos_count, 1, -1)
    return mags * signs


def _check_symmetric(M):
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ShapeError("M must be square")
    if not np.array_equal(M, M.T):
        raise ValueError("M must be exactly symmetric")
    return M


def bunch_parlett_factor_device(Mt, thresh=None):
    """Factor a device-resident symmetric M (torch float64, n x n, either
    storage order) in place of the reference's bunch_parlett_factor.
    Returns (G (torch, shape (n, n) holding G column-major: row c = column
    c), signs (numpy int8), perm (numpy int64), p)."""
    import torch

    require_cuda()
    n = Mt.shape[0]
    if Mt.dim() != 2 or Mt.shape[1] != n:
        raise ShapeError("M must be square")
    Mt = Mt.contiguous()
    if thresh is None:
        thresh = -1.0  # n eps ||M||_F, computed by the library on the device
    L = _lib.load()
    size = ctypes.c_size_t(0)
    _lib.check(L.hsvd_bp_workspace_size(n, ctypes.byref(size)))
    dev = Mt.device
    ws = torch.empty(size.value, dtype=torch.uint8, device=dev)
    Gt = torch.empty((n, n), dtype=torch.float64, device=dev)
    signs = torch.empty(n, dtype=torch.int8, device=dev)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    p = ctypes.c_int64(0)
    stage = ctypes.c_int64(-1)
    st = L.hsvd_bp_factor(ptr(Mt), n, n, float(thresh), ptr(Gt), n, ptr(signs), ptr(perm),
                          ctypes.byref(p), ctypes.byref(stage), ptr(ws), size.value,
                          stream_handle())
    _lib.check(st)
    return Gt, signs.cpu().numpy(), perm.cpu().numpy(), int(p.value)


def bunch_parlett_factor(M):
    """Factor a symmetric M as G J G^T with G of full column rank
    (factory.py:270-282): complete (Bunch-Parlett) pivoting in double-double
    on the GPU, +1 columns first.  Bit-identical to the reference."""
    import torch

    M = _check_symmetric(M)
    n = M.shape[0]
    thresh = n * EPS * np.linalg.norm(M, "fro")  # the reference's threshold
    require_cuda()
    Mt = torch.from_numpy(np.ascontiguousarray(M)).cuda()
    Gt, signs, perm, p = bunch_parlett_factor_device(Mt, thresh)
    G = np.asfortranarray(Gt.cpu().numpy().T)
    return FactorPair(G, SignatureVector.from_p(n, p), perm)


def eigvalsh(M, cfg=None):
    """Eigenvalues of a symmetric M, ascending: Bunch-Parlett on the GPU,
    then the HSVD of (G, J) (lambda = sigma^2 j; the pipeline of
    test_factory.py:134-139)."""
    from .solver import drive

    pair = bunch_parlett_factor(M)
    res = drive(pair.G, pair.J, cfg)
    return np.sort(res.lam)


def qr_shorten(G):
    """Householder QR of a tall factor (factory.py:300-334): G = Q R with R's
    diagonal positive, on the GPU (hsvd_qr_shorten).  The HSVD of R then
    gives the HSVD of G after premultiplying U by Q.  Returns (R, Q)."""
    import torch

    from .linalg import as_factor

    G = as_factor(G)
    n, r = G.shape
    if n <= r:
        raise ShapeError("qr_shorten needs n > r")
    require_cuda()
    L = _lib.load()
    size = ctypes.c_size_t(0)
    _lib.check(L.hsvd_qr_workspace_size(n, r, ctypes.byref(size)))
    Gt = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()  # row c = column c
    ws = torch.empty(size.value, dtype=torch.uint8, device=Gt.device)
    Rt = torch.empty((r, r), dtype=torch.float64, device=Gt.device)
    Qt = torch.empty((r, n), dtype=torch.float64, device=Gt.device)
    bad = ctypes.c_int64(-1)
    st = L.hsvd_qr_shorten(ptr(Gt), n, r, n, ptr(Rt), r, ptr(Qt), n, ctypes.byref(bad), ptr(ws),
                           size.value, stream_handle())
    if st == _lib.HSVD_RANK_DEFICIENT:
        from .errors import RankDeficiencyError
        raise RankDeficiencyError(f"column {bad.value} is dependent" if bad.value >= 0
                                  else _lib.last_error())
    _lib.check(st)
    return (np.asfortranarray(Rt.cpu().numpy().T), np.asfortranarray(Qt.cpu().numpy().T))


def _generate_dd_device(lam, rng, identity_q=False, chunk=64):
    """M = Q diag(lam) Q^T in double-double on the device (factory.py:79-101):
    the n - 1 reflector vectors are the reference's rng.standard_normal(n)
    draws, streamed to the device in chunks.  Returns (Mh, Ml) torch (n, n)."""
    import torch

    require_cuda()
    L = _lib.load()
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    n = lam.shape[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    Mh = torch.empty((n, n), dtype=torch.float64, device=dev)
    Ml = torch.empty((n, n), dtype=torch.float64, device=dev)
    lam_t = torch.from_numpy(lam).to(dev)
    s = stream_handle()
    _lib.check(L.hsvd_gen_init(ptr(lam_t), n, ptr(Mh), ptr(Ml), s))
    if identity_q:
        return Mh, Ml
    size = ctypes.c_size_t(0)
    _lib.check(L.hsvd_gen_workspace_size(n, ctypes.byref(size)))
    ws = torch.empty(size.value, dtype=torch.uint8, device=dev)
    left = n - 1
    while left > 0:
        cnt = min(chunk, left)
        V = np.stack([rng.standard_normal(n) for _ in range(cnt)])
        Vt = torch.from_numpy(V).to(dev)
        _lib.check(L.hsvd_gen_reflect(ptr(Mh), ptr(Ml), n, ptr(Vt), cnt, ptr(ws), size.value, s))
        left -= cnt
    _lib.check(L.hsvd_gen_finish(ptr(Mh), ptr(Ml), n, s))
    return Mh, Ml


def generate_symmetric(spec, eigenvalues=None, identity_q=False):
    """Generate (M, lambda_true) (factory.py:104-114): M exactly symmetric
    with the drawn (or given) spectrum, built in double-double on the GPU
    and rounded to float64; bit-identical to the reference."""
    rng = np.random.default_rng(spec.seed)
    lam = draw_spectrum(spec, rng) if eigenvalues is None else \
        np.asarray(eigenvalues, dtype=np.float64)
    Mh, Ml = _generate_dd_device(lam, rng, identity_q)
    M = (Mh + Ml).cpu().numpy()
    return M, np.sort(lam)


def generate_factor_pair(spec, identity_q=False):
    """Full pipeline (factory.py:285-297): spectrum -> M -> (G, J), chained in
    double-double on the GPU (the factorization consumes the unrounded M)."""
    rng = np.random.default_rng(spec.seed)
    lam = draw_spectrum(spec, rng)
    Mh, Ml = _generate_dd_device(lam, rng, identity_q)
    n = lam.shape[0]
    Mh_np = Mh.cpu().numpy()
    thresh = n * EPS * np.linalg.norm(Mh_np, "fro")
    L = _lib.load()
    import torch

    size = ctypes.c_size_t(0)
    _lib.check(L.hsvd_bp_workspace_size(n, ctypes.byref(size)))
    ws = torch.empty(size.value, dtype=torch.uint8, device=Mh.device)
    Gt = torch.empty((n, n), dtype=torch.float64, device=Mh.device)
    signs = torch.empty(n, dtype=torch.int8, device=Mh.device)
    perm = torch.empty(n, dtype=torch.int64, device=Mh.device)
    p = ctypes.c_int64(0)
    stage = ctypes.c_int64(-1)
    _lib.check(L.hsvd_bp_factor_dd(ptr(Mh), ptr(Ml), n, n, float(thresh), ptr(Gt), n,
                                   ptr(signs), ptr(perm), ctypes.byref(p), ctypes.byref(stage),
                                   ptr(ws), size.value, stream_handle()))
    G = np.asfortranarray(Gt.cpu().numpy().T)
    factor = FactorPair(G, SignatureVector.from_p(n, int(p.value)), perm.cpu().numpy())
    M = (Mh + Ml).cpu().numpy()
    return TestBundle(M, np.sort(lam), factor, spec)
