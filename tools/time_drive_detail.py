"""Host-side stages of drive_device (allocation, C call, marshalling)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402
from paper_1008_1371_b200 import _device, _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = np.random.default_rng(0).standard_normal((n, n))
J = H.SignatureVector.from_p(n, n // 2)
G0 = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
cfg = H.SolverConfig(mode="block", block_cols=32)
L = _lib.load()
keep = []
for it in range(5):
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    Gt = G0.clone()
    r = n
    Vt = torch.empty((r, r), dtype=torch.float64, device="cuda")
    sigma = torch.empty(r, dtype=torch.float64, device="cuda")
    lam = torch.empty(r, dtype=torch.float64, device="cuda")
    ccfg = cfg.to_c()
    wsb = L.hsvd_drive_workspace_size(n, r, ccfg)
    ws = torch.empty(max(int(wsb), 1), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    res = _lib.HsvdResultC()
    tele = (_lib.HsvdTelemetryC * 30)()
    signs = np.ascontiguousarray(J.signs, dtype=np.int8)
    st = L.hsvd_drive(_device.ptr(Gt), n, r, n, _device.ptr(Vt), r,
                      signs.ctypes.data_as(ctypes.c_void_p), J.p, ccfg,
                      _device.ptr(sigma), _device.ptr(lam), _device.ptr(ws),
                      int(wsb), res, tele, _device.stream_handle())
    T.append(time.perf_counter())
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    keep.append((Gt, Vt))
    if len(keep) > 2:
        keep.pop(0)
    d = np.diff(T) * 1e3
    print(f"it {it}: alloc {d[0]:.1f} ms, hsvd_drive {d[1]:.1f} (setup {res.setup_ms:.1f} "
          f"sweeps {res.sweeps_ms:.1f} finish {res.finish_ms:.1f}), tail sync {d[2]:.1f}", flush=True)
