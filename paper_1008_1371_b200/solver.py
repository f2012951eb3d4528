"""One-sided hyperbolic Jacobi driver -- the drop-in for hjsvd.drive
(/root/reference/pkg/src/hjsvd/solver.py:179-269).

The host does validation and result marshalling only; the whole quasi-sweep
loop (steps, convergence test, sort) runs on the device inside
libhsvd_b200's hsvd_drive.  Two modes:

* ``mode="pointwise"`` (default): the reference's algorithm, bit-identical
  results (sigma, U, lam, V^{-T}, sweeps, rotations, skips, telemetry).
* ``mode="block"``: block-column pairs with FP64 tensor-core Gram/update
  GEMMs; sigma agrees with the reference to ~1e-13 relative, sweeps are
  block sweeps (reported next to the reference's).
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .errors import DefinitenessLostError, RankDeficiencyError, ShapeError
from .linalg import DEFAULT_CHUNK, EPS, SignatureVector, as_factor
from .strategies import StepperState, stepper_init  # noqa: F401

_STOP = {0: "orthogonal", 1: "quadratic", 2: "max_sweeps"}


@dataclass
class DiagonalPackageVector:
    """Per-position packages (d, rho, j) (solver.py:26-43)."""

    d: np.ndarray
    rho: np.ndarray
    jsign: np.ndarray
    p: int

    def copy(self):
        return DiagonalPackageVector(self.d.copy(), self.rho.copy(),
                                     self.jsign.copy(), self.p)


@dataclass
class SolverConfig:
    """SolverConfig (solver.py:46-64) with the same fields and defaults, plus
    the B200 knobs (mode, block_cols, inner_ordering, use_graph).  workers
    is accepted and ignored: the device result does not depend on it."""

    max_sweeps: int = 30
    eps: float = EPS
    teps: float = None
    accumulate_v: bool = True
    use_rel_orth_skip: bool = True
    chunk: int = DEFAULT_CHUNK
    workers: int = 1
    schedule: str = "modulus"
    sort: bool = True
    mode: str = "pointwise"
    block_cols: int = 32
    inner_ordering: str = "full"
    use_graph: bool = True
    profile: bool = False
    #: block mode 2x2 rotation: "fast" (plain fp64) or "dd" (the reference's
    #: double-double rotation_tc, _kernels.py:128-173)
    block_rotation: str = "fast"
    #: block mode: passes of the inner ordering per step; 0 = auto (2 in the
    #: dense sweeps, 1 once a sweep rotates < 5 % of its visits)
    inner_passes: int = 0
    #: block mode on one GPU: 2 = two half-slot streams (inner passes overlap
    #: GEMMs), 1 = one stream
    block_streams: int = 2

    def __post_init__(self):
        if self.teps is None:
            self.teps = math.sqrt(self.eps) / 2.0
        if self.schedule not in ("modulus", "row-cyclic"):
            raise ValueError(f"unknown schedule {self.schedule!r}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.mode not in ("pointwise", "block"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.inner_ordering not in ("oriented", "full"):
            raise ValueError(f"unknown inner_ordering {self.inner_ordering!r}")
        if self.block_cols not in (16, 32):
            raise ValueError("block_cols must be 16 or 32")
        if self.block_streams not in (1, 2):
            raise ValueError("block_streams must be 1 or 2")
        if self.inner_passes < 0:
            raise ValueError("inner_passes must be >= 0 (0: auto)")
        if self.block_rotation not in ("fast", "dd"):
            raise ValueError(f"unknown block_rotation {self.block_rotation!r}")

    def to_c(self):
        c = _lib.HsvdConfigC()
        c.max_sweeps = int(self.max_sweeps)
        c.eps = float(self.eps)
        c.teps = float(self.teps)
        c.accumulate_v = int(bool(self.accumulate_v))
        c.use_skip = int(bool(self.use_rel_orth_skip))
        c.chunk = int(self.chunk)
        c.schedule = (_lib.SCHEDULE_ROW_CYCLIC if self.schedule == "row-cyclic"
                      else _lib.SCHEDULE_MODULUS)
        c.sort = int(bool(self.sort))
        c.mode = _lib.MODE_BLOCK if self.mode == "block" else _lib.MODE_POINTWISE
        c.block_cols = int(self.block_cols)
        c.inner_full = int(self.inner_ordering == "full")
        c.use_graph = int(bool(self.use_graph))
        c.profile = int(bool(self.profile))
        c.block_rotation = int(self.block_rotation == "fast")
        c.inner_passes = int(self.inner_passes)
        c.block_streams = int(self.block_streams)
        return c


@dataclass
class HsvdResult:
    """HsvdResult (solver.py:67-77).  Arrays are numpy for numpy input and
    torch CUDA tensors for CUDA-tensor input."""

    sigma: object
    U: object
    lam: object
    Vinv_t: object = None
    sweeps_used: int = 0
    stop_reason: str = "max_sweeps"
    rotations: int = 0
    skips: int = 0
    telemetry: list = field(default_factory=list)
    #: B200 extras: device time of each sweep (ms) and kernel launches
    sweep_gpu_ms: list = field(default_factory=list)
    gpu_launches: int = 0
    host_phase_ms: dict = field(default_factory=dict)
    kernel_profile: dict = field(default_factory=dict)


def precompute(G, J, chunk=DEFAULT_CHUNK):
    """Initial packages (solver.py:80-94); norms computed on the device."""
    G = as_factor(G)
    n, r = G.shape
    if len(J) != r:
        raise ShapeError("signature length must match the column count")
    d, bad = _device.precompute(G, chunk)
    if bad >= 0:
        raise RankDeficiencyError(f"column {bad} has zero norm")
    return DiagonalPackageVector(d, np.arange(r, dtype=np.int64),
                                 J.signs.astype(np.int64), J.p)


def sort_diagonal(D, p=None):
    """Stable two-segment sort of the packages, on the device (solver.py:97-110)."""
    if p is None:
        p = D.p
    _device.sort_diagonal(D.d, D.rho, D.jsign, p)
    return D


def check_convergence(C):
    """Or-reduce the per-block codes into a stop decision (solver.py:113-121).
    (The solver itself reduces the codes on the device.)"""
    code = int(np.bitwise_or.reduce(np.asarray(C))) if len(C) else 0
    assert code != 0b10, "convergence code (10)2 must be unreachable"
    if code == 0b00:
        return "stop_orthogonal"
    if code == 0b01:
        return "stop_quadratic"
    return "continue"


def jacobi_step(G, Vinv_t, D, S, C, cfg=None):
    """One parallel step on the device, then advance (solver.py:159-176).
    Mutates G, Vinv_t, D, C and S in place; returns (rotations, skips, max|t|)."""
    if cfg is None:
        cfg = SolverConfig()
    stats = _device.step_blocks(G, Vinv_t, D.d, D.rho, D.jsign, S.iblk, S.jblk,
                                C, cfg)
    _device.advance_stepper(S.ip, S.jp, S.iblk, S.jblk, S.r)
    return stats


def drive_device(Gt, J, cfg=None, n=None):
    """Solve with the factor already in HBM.

    Gt: CUDA float64 tensor of shape (r, n), C-contiguous -- i.e. the n x r
    column-major factor G.  It is OVERWRITTEN by U (same layout).  Returns
    an HsvdResult whose arrays are CUDA tensors (sigma, lam: (r,);
    U: the (r, n) tensor Gt; Vinv_t: (r, r) column-major, i.e. Vinv_t[c]
    is column c of V^{-T})."""
    if cfg is None:
        cfg = SolverConfig()
    if Gt.dtype != torch.float64 or not Gt.is_cuda or not Gt.is_contiguous():
        raise ValueError("Gt must be a contiguous float64 CUDA tensor (r, n)")
    r, n = Gt.shape
    if len(J) != r:
        raise ShapeError("signature length must match the column count")
    if r % 2 != 0:
        raise ShapeError("r must be even; use border() first")
    if n < r:
        raise ShapeError("G must have n >= r")
    dev = Gt.device
    L = _lib.load()
    ccfg = cfg.to_c()
    Vt = (torch.empty((r, r), dtype=torch.float64, device=dev)
          if cfg.accumulate_v else None)
    sigma = torch.empty(r, dtype=torch.float64, device=dev)
    lam = torch.empty(r, dtype=torch.float64, device=dev)
    wsb = L.hsvd_drive_workspace_size(n, r, ccfg)
    ws = torch.empty(max(int(wsb), 1), dtype=torch.uint8, device=dev)
    res = _lib.HsvdResultC()
    tele = (_lib.HsvdTelemetryC * max(int(cfg.max_sweeps), 1))()
    signs = np.ascontiguousarray(J.signs, dtype=np.int8)
    st = L.hsvd_drive(_device.ptr(Gt), n, r, n, _device.ptr(Vt), r,
                      signs.ctypes.data_as(_device.ctypes.c_void_p), J.p, ccfg,
                      _device.ptr(sigma), _device.ptr(lam), _device.ptr(ws),
                      int(wsb), res, tele, _device.stream_handle())
    _lib.check(st, tuple(res.err))
    telemetry = [(int(tele[s].sweep), int(tele[s].rotations),
                  int(tele[s].skips), float(tele[s].max_t))
                 for s in range(res.sweeps_used)]
    names = (("step", "inner", "update", "sweep_end") if cfg.mode == "pointwise"
             else ("gram", "inner", "update", "sweep_end"))
    prof = ({names[k]: {"ms": float(res.kernel_ms[k]),
                        "launches": int(res.kernel_launches[k])}
             for k in range(4) if res.kernel_launches[k]} if cfg.profile else {})
    return HsvdResult(sigma, Gt, lam, Vt, int(res.sweeps_used),
                      _STOP[int(res.stop_reason)], int(res.rotations),
                      int(res.skips), telemetry,
                      [float(tele[s].gpu_ms) for s in range(res.sweeps_used)],
                      int(res.launches),
                      {"setup": float(res.setup_ms), "sweeps": float(res.sweeps_ms),
                       "finish": float(res.finish_ms)},
                      prof)


def drive(G, J, cfg=None):
    """Full HSVD of the factor pair (G, J) (solver.py:179-269).

    numpy (or array-like) G: the caller's array is never mutated; results
    are numpy arrays in the original column order, exactly as the
    reference returns them.  A CUDA float64 tensor G of shape (n, r) is
    accepted too (results stay on the device)."""
    if cfg is None:
        cfg = SolverConfig()
    if isinstance(G, torch.Tensor) and G.is_cuda:
        if G.dim() != 2:
            raise ShapeError("G must be a matrix")
        # always a fresh buffer: drive_device overwrites it with U, and the
        # caller's G is never mutated (solver.py:188).  (.t().contiguous()
        # would alias a column-major float64 G.)
        Gt = G.detach().to(torch.float64).t().clone(memory_format=torch.contiguous_format)
        res = drive_device(Gt, J, cfg)
        res.U = res.U.t()
        if res.Vinv_t is not None:
            res.Vinv_t = res.Vinv_t.t()
        return res
    # as_factor (linalg.py:58-65) without its host-side finiteness scan: the
    # library checks the factor on the device before the solve (ValueError)
    G = np.asfortranarray(G, dtype=np.float64)
    if G.ndim != 2:
        raise ShapeError("G must be a matrix")
    n, r = G.shape
    if len(J) != r:
        raise ShapeError("signature length must match the column count")
    if r % 2 != 0:
        raise ShapeError("r must be even; use border() first")
    if n < r:
        raise ShapeError("G must have n >= r")
    dev = _device.require_cuda()
    Gt = _device.colmajor_to_device(G, dev)
    res = drive_device(Gt, J, cfg)
    # results land in page-locked host memory (a pageable device->host copy
    # runs at a fraction of the link rate); the numpy arrays keep it alive
    res.U = _device.device_to_colmajor_pinned(res.U)
    if res.Vinv_t is not None:
        res.Vinv_t = _device.device_to_colmajor_pinned(res.Vinv_t)
    res.sigma = res.sigma.cpu().numpy()
    res.lam = res.lam.cpu().numpy()
    return res


def recover_V(Vinv_t, J):
    """V = J V^{-T} J (solver.py:272-275)."""
    if isinstance(Vinv_t, torch.Tensor):
        s = torch.as_tensor(J.signs.astype(np.float64), device=Vinv_t.device)
        return s[:, None] * Vinv_t * s[None, :]
    s = J.signs.astype(np.float64)
    return s[:, np.newaxis] * Vinv_t * s[np.newaxis, :]


@dataclass(frozen=True)
class BorderInfo:
    """How a factor was embedded (solver.py:278-286)."""

    orig_n: int
    orig_r: int
    target_n: int
    target_r: int
    synthetic_col: int = -1


def border(G, J, target_r, target_n):
    """Embed G top-left into a target_n x target_r factor (solver.py:289-320,
    PAPER.md:599-642).  Host-side data preparation."""
    G = as_factor(G)
    n, r = G.shape
    if target_r not in (r, r + 1) or target_r % 2 != 0:
        raise ShapeError("target_r must be r or r+1 and even")
    need_col = target_r == r + 1
    min_n = n + 1 if need_col else n
    if target_n < max(min_n, target_r):
        raise ShapeError("target_n too small for the bordered factor")
    G2 = np.zeros((target_n, target_r), order="F")
    p = J.p
    if need_col:
        G2[:n, :p] = G[:, :p]
        G2[n, p] = 1.0
        G2[:n, p + 1:] = G[:, p:]
        return G2, SignatureVector.from_p(target_r, p + 1), BorderInfo(
            n, r, target_n, target_r, p)
    G2[:n, :r] = G
    return G2, SignatureVector.from_p(target_r, p), BorderInfo(
        n, r, target_n, target_r, -1)


def strip_bordered(result, info):
    """Drop the synthetic column and padding rows (solver.py:323-341)."""
    cols = np.arange(info.target_r)
    if info.synthetic_col >= 0:
        cols = np.delete(cols, info.synthetic_col)
    Vinv_t = result.Vinv_t
    if Vinv_t is not None:
        Vinv_t = np.asfortranarray(np.asarray(Vinv_t)[np.ix_(cols, cols)])
    return HsvdResult(
        sigma=np.asarray(result.sigma)[cols],
        U=np.asfortranarray(np.asarray(result.U)[: info.orig_n, :][:, cols]),
        lam=np.asarray(result.lam)[cols],
        Vinv_t=Vinv_t,
        sweeps_used=result.sweeps_used,
        stop_reason=result.stop_reason,
        rotations=result.rotations,
        skips=result.skips,
        telemetry=result.telemetry,
    )
