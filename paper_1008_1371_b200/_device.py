"""Device plumbing: torch owns HBM buffers and streams, libhsvd_b200 does
the work.  A column-major n x r float64 matrix lives on the device as a
C-contiguous torch tensor of shape (r, n) (row c = column c), so the
leading dimension is n and no transposition ever happens on the device."""

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import DefinitenessLostError


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1008_1371_b200 needs a CUDA device (sm_100a); there is no "
            "CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


_POOL = None
_STAGE_MIN = 32 << 20  # bytes: below this a direct pageable copy is as fast


def _pool():
    global _POOL
    if _POOL is None:
        import concurrent.futures
        import os
        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    return _POOL


def colmajor_to_device(G, dev):
    """numpy (n, r) any order -> device (r, n) contiguous = column-major G.

    Large factors are staged through page-locked memory in chunks: host
    threads copy chunk k (numpy releases the GIL) while the DMA engine moves
    chunk k-1 at link rate (a pageable copy runs at a fraction of it)."""
    src = np.asarray(G, dtype=np.float64).T  # (r, n): C-contiguous for F-order G
    if src.nbytes < _STAGE_MIN or not src.flags.c_contiguous:
        host = np.ascontiguousarray(src)
        if not host.flags.writeable:  # torch.from_numpy wants a writable array
            host = host.copy()
        return torch.from_numpy(host).to(dev, non_blocking=False)
    out = torch.empty(src.shape, dtype=torch.float64, device=dev)
    host = torch.empty(src.shape, dtype=torch.float64, pin_memory=True)
    hv = host.numpy()
    rows = src.shape[0]
    nch = 16
    bounds = [rows * k // nch for k in range(nch + 1)]
    futs = [_pool().submit(np.copyto, hv[bounds[k]:bounds[k + 1]], src[bounds[k]:bounds[k + 1]])
            for k in range(nch)]
    for k in range(nch):
        futs[k].result()
        a, b = bounds[k], bounds[k + 1]
        if b > a:
            out[a:b].copy_(host[a:b], non_blocking=True)
    return out


def device_to_colmajor(Gt):
    """device (r, n) -> numpy Fortran-ordered (n, r)."""
    return np.asfortranarray(Gt.cpu().numpy().T)


def device_to_colmajor_pinned(Gt):
    """device (r, n) -> numpy Fortran-ordered (n, r) backed by page-locked
    host memory (torch's caching host allocator), copied at link rate."""
    host = torch.empty(Gt.shape, dtype=Gt.dtype, pin_memory=True)
    host.copy_(Gt, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy().T


def _vec(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _i64(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).to(dev)


# ---- reference-kernel mirrors ------------------------------------------


def dot_chunked(x, y, chunk):
    dev = require_cuda()
    L = _lib.load()
    xd, yd = _vec(x, dev), _vec(y, dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(L.hsvd_dot_chunked(ptr(xd), ptr(yd), x.shape[0], chunk, ptr(out),
                                  stream_handle()))
    return float(out.item())


def fused_pair_update(x, y, t, c, s, chunk):
    dev = require_cuda()
    L = _lib.load()
    xd, yd = _vec(x, dev), _vec(y, dev)
    n = x.shape[0]
    _lib.check(L.hsvd_fused_pair_update(ptr(xd), ptr(yd), n, t, c, s,
                                        stream_handle()))
    out = torch.empty(2, dtype=torch.float64, device=dev)
    _lib.check(L.hsvd_dot_chunked(ptr(xd), ptr(xd), n, chunk, ptr(out[0:1]),
                                  stream_handle()))
    _lib.check(L.hsvd_dot_chunked(ptr(yd), ptr(yd), n, chunk, ptr(out[1:2]),
                                  stream_handle()))
    x[...] = xd.cpu().numpy()
    y[...] = yd.cpu().numpy()
    o = out.cpu().numpy()
    return float(o[0]), float(o[1])


def rotation_batch(a_ii, a_jj, a_ij, hyp):
    dev = require_cuda()
    L = _lib.load()
    m = a_ii.shape[0]
    A, B, Cd = _vec(a_ii, dev), _vec(a_jj, dev), _vec(a_ij, dev)
    H = _i64(hyp, dev)
    t = torch.empty(m, dtype=torch.float64, device=dev)
    c = torch.empty(m, dtype=torch.float64, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(L.hsvd_rotation_batch(ptr(A), ptr(B), ptr(Cd), ptr(H), m, ptr(t),
                                     ptr(c), ptr(bad), stream_handle()))
    return t.cpu().numpy(), c.cpu().numpy(), int(bad.item())


def precompute(G, chunk):
    """d[k] = dot_chunked(g_k, g_k) on the device; returns (d, first_zero)."""
    dev = require_cuda()
    L = _lib.load()
    n, r = G.shape
    Gt = colmajor_to_device(G, dev)
    d = torch.empty(r, dtype=torch.float64, device=dev)
    fz = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(L.hsvd_precompute(ptr(Gt), n, r, n, chunk, ptr(d), ptr(fz),
                                 stream_handle()))
    return d.cpu().numpy(), int(fz.item())


def sort_diagonal(d, rho, jsign, p):
    """In-place stable two-segment sort of numpy package arrays on the device."""
    dev = require_cuda()
    L = _lib.load()
    r = d.shape[0]
    dd, rr, jj = _vec(d, dev), _i64(rho, dev), _i64(jsign, dev)
    ws = torch.empty(24 * max(r, 1), dtype=torch.uint8, device=dev)
    _lib.check(L.hsvd_sort_diagonal(ptr(dd), ptr(rr), ptr(jj), r, p, ptr(ws),
                                    stream_handle()))
    d[...] = dd.cpu().numpy()
    rho[...] = rr.cpu().numpy()
    jsign[...] = jj.cpu().numpy()


def advance_stepper(ip, jp, iblk, jblk, r):
    dev = require_cuda()
    L = _lib.load()
    arrs = [_i64(a, dev) for a in (ip, jp, iblk, jblk)]
    _lib.check(L.hsvd_advance_stepper(*[ptr(a) for a in arrs], ip.shape[0], r,
                                      stream_handle()))
    for host, d in zip((ip, jp, iblk, jblk), arrs):
        host[...] = d.cpu().numpy()


def step_blocks(G, V, d, rho, jsign, iblk, jblk, C, cfg):
    """One step of all slots (_kernels.step_blocks over [0, b)) on numpy
    arrays, in place.  Returns (rotations, skips, max|t|)."""
    dev = require_cuda()
    L = _lib.load()
    n, r = G.shape
    b = iblk.shape[0]
    Gt = colmajor_to_device(G, dev)
    Vt = colmajor_to_device(V, dev) if V is not None else None
    dd, rr, jj = _vec(d, dev), _i64(rho, dev), _i64(jsign, dev)
    ib, jb = _i64(iblk, dev), _i64(jblk, dev)
    Cd = torch.from_numpy(np.ascontiguousarray(C, dtype=np.uint8)).to(dev)
    rotk = torch.zeros(b, dtype=torch.int32, device=dev)
    skipk = torch.zeros(b, dtype=torch.int32, device=dev)
    maxt = torch.zeros(b, dtype=torch.float64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    out = torch.zeros(8, dtype=torch.int64, device=dev)
    s = stream_handle()
    rv = V.shape[0] if V is not None else 0
    _lib.check(L.hsvd_step_blocks(
        ptr(Gt), n, n, ptr(Vt), rv, rv, ptr(dd), ptr(rr), ptr(jj), None, None,
        ptr(ib), ptr(jb), r, ptr(Cd), 0, b, cfg.eps, cfg.teps,
        int(cfg.use_rel_orth_skip), cfg.chunk, 0, ptr(rotk), ptr(skipk),
        ptr(maxt), ptr(err), s))
    _lib.check(L.hsvd_reduce_sweep(ptr(Cd), 0, ptr(rotk), ptr(skipk), ptr(maxt),
                                   b, ptr(out), 0, s))
    e = int(err.item())
    if e != -1:
        w = e & ((1 << 64) - 1)
        raise DefinitenessLostError(w >> 42, (w >> 21) & ((1 << 21) - 1),
                                    w & ((1 << 21) - 1))
    G[...] = device_to_colmajor(Gt)
    if V is not None:
        V[...] = device_to_colmajor(Vt)
    d[...] = dd.cpu().numpy()
    C[...] = Cd.cpu().numpy()
    o = out.cpu().numpy()
    max_t = float(np.array([o[3]], dtype=np.int64).view(np.float64)[0])
    return int(o[1]), int(o[2]), max_t
