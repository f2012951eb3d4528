"""Block-mode HSVD sharded over GPUs.

The reference runs the slots of one parallel step on worker threads in
contiguous ranges (_run_ranges, /root/reference/pkg/src/hjsvd/solver.py:124-156)
and its result does not depend on the split (test_solver.py:167-173).  Here
the ranges are GPUs: shard g owns slots [g*S/N, (g+1)*S/N) of the S = r/(2b)
block slots and keeps their block columns of G and V^{-T} in its own HBM.
libhsvd_b200's hsvd_drive_sharded moves one block column per step to a ring
neighbour (NCCL send/recv), all-gathers the norms at the end of each sweep,
sorts them identically on every shard and redistributes the columns with a
grouped all-to-all; the stop decision is all-reduced, so every rank leaves
the sweep loop together.

* ``drive_sharded(G, J, cfg, comm)`` -- one process per GPU (torchrun):
  every rank passes the full factor and gets back its own columns
  (``ShardedResult``); ``gather_result`` assembles the full HsvdResult.
* ``drive_local_shards(G, J, cfg, nshards)`` -- one process drives all
  shards (streams on the current device, peer copies instead of NCCL): the
  same plan, exchanges, redistribution and kernels, runnable on one GPU.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .errors import ShapeError
from .solver import _STOP, HsvdResult, SolverConfig


@dataclass
class ShardedResult:
    """One shard's part of an HsvdResult: the columns it holds after the
    final sweep.  ``cols[k]`` is the ORIGINAL column index of local column k;
    U (n, cols) / Vinv_t (r, cols) are column slices (device tensors of
    shape (cols, n) / (cols, r) in the library's column-major convention are
    kept in ``U_t`` / ``Vinv_t_t``)."""

    shard: int
    nshards: int
    cols: np.ndarray
    sigma: torch.Tensor
    lam: torch.Tensor
    U_t: torch.Tensor
    Vinv_t_t: torch.Tensor = None
    sweeps_used: int = 0
    stop_reason: str = "max_sweeps"
    rotations: int = 0
    skips: int = 0
    telemetry: list = field(default_factory=list)
    sweep_gpu_ms: list = field(default_factory=list)
    gpu_launches: int = 0
    host_phase_ms: dict = field(default_factory=dict)
    #: profile mode: device ms / launches per kernel class of sweep 0 on the
    #: first local shard (gram, inner, update)
    kernel_profile: dict = field(default_factory=dict)


class ShardComm:
    """The sharded solver's NCCL communicator, bootstrapped over an
    initialised torch.distributed group (the id is broadcast with it)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        L = _lib.load()
        buf = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _lib.check(L.hsvd_comm_unique_id(buf))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        ctypes.memmove(buf, obj[0], 128)
        self.handle = ctypes.c_void_p()
        _lib.check(L.hsvd_comm_init(buf, self.world, self.rank, ctypes.byref(self.handle)))

    def close(self):
        if self.handle:
            _lib.load().hsvd_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_cfg(cfg, r):
    if cfg is None:
        cfg = SolverConfig(mode="block")
    if cfg.mode != "block":
        raise NotImplementedError("the sharded solver runs block mode only")
    if r % 2:
        raise ShapeError("r must be even; use border() first")
    return cfg


def _factor_on(G, dev):
    """(r, n) column-major device copy of the factor (numpy or CUDA tensor)."""
    if isinstance(G, torch.Tensor):
        if G.dim() != 2:
            raise ShapeError("G must be a matrix")
        return G.detach().to(device=dev, dtype=torch.float64).t().contiguous()
    return _device.colmajor_to_device(G, dev)


def _run(comm, nshards, shard_ids, devices, Gts, n, r, J, cfg):
    L = _lib.load()
    ccfg = cfg.to_c()
    nl = len(shard_ids)
    outs = []
    for g, dev in zip(shard_ids, devices):
        cols = int(L.hsvd_shard_columns(r, cfg.block_cols, nshards, g))
        if cols < 0:
            raise NotImplementedError(
                f"r={r}, block_cols={cfg.block_cols} does not shard over {nshards} GPUs "
                "(need r/(2b) >= shards)")
        wsb = int(L.hsvd_sharded_workspace_size(n, r, nshards, g, ccfg))
        d = torch.device("cuda", dev)
        outs.append({
            "cols": np.empty(cols, np.int64),
            "U": torch.empty((cols, n), dtype=torch.float64, device=d),
            "V": (torch.empty((cols, r), dtype=torch.float64, device=d)
                  if cfg.accumulate_v else None),
            "sigma": torch.empty(cols, dtype=torch.float64, device=d),
            "lam": torch.empty(cols, dtype=torch.float64, device=d),
            "ws": torch.empty(max(wsb, 1), dtype=torch.uint8, device=d),
            "wsb": wsb,
        })
    P = ctypes.c_void_p
    arr = lambda xs: (P * nl)(*[P(x) for x in xs])  # noqa: E731
    ids = (ctypes.c_int32 * nl)(*shard_ids)
    devs = (ctypes.c_int32 * nl)(*devices)
    res = _lib.HsvdResultC()
    tele = (_lib.HsvdTelemetryC * max(int(cfg.max_sweeps), 1))()
    signs = np.ascontiguousarray(J.signs, dtype=np.int8)
    for dev in set(devices):
        torch.cuda.synchronize(dev)
    st = L.hsvd_drive_sharded(
        comm.handle if comm is not None else None, nshards, nl, ids, devs,
        arr([g.data_ptr() for g in Gts]), n, r, n,
        signs.ctypes.data_as(P), J.p, ccfg,
        arr([o["U"].data_ptr() for o in outs]),
        arr([o["V"].data_ptr() if o["V"] is not None else 0 for o in outs]),
        arr([o["cols"].ctypes.data for o in outs]),
        arr([o["sigma"].data_ptr() for o in outs]),
        arr([o["lam"].data_ptr() for o in outs]),
        arr([o["ws"].data_ptr() for o in outs]),
        (ctypes.c_int64 * nl)(*[o["wsb"] for o in outs]),
        res, tele)
    _lib.check(st, tuple(res.err))
    telemetry = [(int(tele[s].sweep), int(tele[s].rotations), int(tele[s].skips),
                  float(tele[s].max_t)) for s in range(res.sweeps_used)]
    common = dict(sweeps_used=int(res.sweeps_used), stop_reason=_STOP[int(res.stop_reason)],
                  rotations=int(res.rotations), skips=int(res.skips), telemetry=telemetry,
                  sweep_gpu_ms=[float(tele[s].gpu_ms) for s in range(res.sweeps_used)],
                  gpu_launches=int(res.launches),
                  host_phase_ms={"setup": float(res.setup_ms), "sweeps": float(res.sweeps_ms),
                                 "finish": float(res.finish_ms)},
                  kernel_profile=({nm: {"ms": float(res.kernel_ms[k]),
                                        "launches": int(res.kernel_launches[k])}
                                   for k, nm in enumerate(("gram", "inner", "update"))
                                   if res.kernel_launches[k]} if cfg.profile else {}))
    return [ShardedResult(shard=g, nshards=nshards, cols=o["cols"], sigma=o["sigma"],
                          lam=o["lam"], U_t=o["U"], Vinv_t_t=o["V"], **common)
            for g, o in zip(shard_ids, outs)]


def drive_sharded(G, J, cfg=None, comm=None):
    """This rank's shard of a block-mode HSVD over ``comm.world`` GPUs.

    Every rank passes the same full factor G (numpy n x r, or a CUDA tensor)
    and returns a ShardedResult with the columns it holds at the end.  The
    call is synchronous (it returns when the solve has finished)."""
    if comm is None:
        raise ValueError("drive_sharded needs a ShardComm (use drive_local_shards "
                         "for one process)")
    n, r = (G.shape[0], G.shape[1])
    dev = _device.require_cuda()
    return drive_sharded_device(_factor_on(G, dev), J, cfg, comm)


def drive_sharded_device(Gt, J, cfg=None, comm=None):
    """drive_sharded on a factor already in HBM: Gt is the (r, n)
    C-contiguous float64 CUDA tensor of the column-major n x r factor (read
    only -- the shard gathers its columns into its own storage)."""
    if comm is None:
        raise ValueError("drive_sharded_device needs a ShardComm")
    if Gt.dtype != torch.float64 or not Gt.is_cuda or not Gt.is_contiguous():
        raise ValueError("Gt must be a contiguous float64 CUDA tensor (r, n)")
    r, n = Gt.shape
    if len(J) != r:
        raise ShapeError("signature length must match the column count")
    if n < r:
        raise ShapeError("G must have n >= r")
    cfg = _check_cfg(cfg, r)
    return _run(comm, comm.world, [comm.rank], [Gt.device.index], [Gt], n, r, J, cfg)[0]


def assemble(parts, n, r, to_numpy=True):
    """Full HsvdResult (original column order) from every shard's part."""
    dev = parts[0].sigma.device
    sigma = torch.empty(r, dtype=torch.float64, device=dev)
    lam = torch.empty(r, dtype=torch.float64, device=dev)
    Ut = torch.empty((r, n), dtype=torch.float64, device=dev)
    with_v = parts[0].Vinv_t_t is not None
    Vt = torch.empty((r, r), dtype=torch.float64, device=dev) if with_v else None
    for pt in parts:
        idx = torch.as_tensor(pt.cols, device=dev)
        sigma[idx] = pt.sigma.to(dev)
        lam[idx] = pt.lam.to(dev)
        Ut[idx] = pt.U_t.to(dev)
        if with_v:
            Vt[idx] = pt.Vinv_t_t.to(dev)
    p0 = parts[0]
    res = HsvdResult(sigma, Ut, lam, Vt, p0.sweeps_used, p0.stop_reason, p0.rotations,
                     p0.skips, p0.telemetry, p0.sweep_gpu_ms, p0.gpu_launches,
                     p0.host_phase_ms)
    if to_numpy:
        torch.cuda.synchronize(dev)
        res.sigma = sigma.cpu().numpy()
        res.lam = lam.cpu().numpy()
        res.U = _device.device_to_colmajor(Ut)
        res.Vinv_t = _device.device_to_colmajor(Vt) if with_v else None
    else:
        res.U = Ut.t()
        res.Vinv_t = Vt.t() if with_v else None
    return res


def gather_result(part, n, r, group=None, to_numpy=True):
    """All-gather every rank's ShardedResult into the full HsvdResult."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    metas = [None] * world
    dist.all_gather_object(metas, (part.shard, part.cols), group=group)
    parts = []
    for g, cols in sorted(metas, key=lambda x: x[0]):
        k = len(cols)
        dev = part.sigma.device
        parts.append(ShardedResult(
            shard=g, nshards=world, cols=cols,
            sigma=torch.empty(k, dtype=torch.float64, device=dev),
            lam=torch.empty(k, dtype=torch.float64, device=dev),
            U_t=torch.empty((k, n), dtype=torch.float64, device=dev),
            Vinv_t_t=(torch.empty((k, r), dtype=torch.float64, device=dev)
                      if part.Vinv_t_t is not None else None),
            sweeps_used=part.sweeps_used, stop_reason=part.stop_reason,
            rotations=part.rotations, skips=part.skips, telemetry=part.telemetry,
            sweep_gpu_ms=part.sweep_gpu_ms, gpu_launches=part.gpu_launches,
            host_phase_ms=part.host_phase_ms))
    for src in range(world):
        for name in ("sigma", "lam", "U_t", "Vinv_t_t"):
            t = getattr(parts[src], name)
            if t is None:
                continue
            if src == part.shard:
                t.copy_(getattr(part, name))
            dist.broadcast(t, src=src, group=group)
    return assemble(parts, n, r, to_numpy)


def drive_local_shards(G, J, cfg=None, nshards=2, devices=None):
    """Block-mode HSVD split into ``nshards`` shards driven by this process
    (one stream per shard on the current device, or on ``devices``).
    Returns the full HsvdResult; numpy in, numpy out."""
    n, r = (G.shape[0], G.shape[1])
    if len(J) != r:
        raise ShapeError("signature length must match the column count")
    cfg = _check_cfg(cfg, r)
    dev = _device.require_cuda()
    if devices is None:
        devices = [dev.index] * nshards
    on = {}
    for d in devices:
        if d not in on:
            on[d] = _factor_on(G, torch.device("cuda", d))
    Gts = [on[d] for d in devices]
    parts = _run(None, nshards, list(range(nshards)), list(devices), Gts, n, r, J, cfg)
    return assemble(parts, n, r, to_numpy=not isinstance(G, torch.Tensor))
