"""Host-side stages of drive(G_numpy, J) at size n (the e2e path)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402
from paper_1008_1371_b200 import _device  # noqa: E402
from paper_1008_1371_b200.linalg import as_factor  # noqa: E402
from tests.golden.inputs import make_case_input  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = make_case_input(n, n, 0, "gauss")
print("input flags: F", G.flags.f_contiguous, "C", G.flags.c_contiguous)
J = H.SignatureVector.from_p(n, n // 2)
dev = torch.device("cuda", 0)
cfg = H.SolverConfig(mode="block")
for it in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    Gf = as_factor(G); t.append(time.perf_counter())
    Gt = _device.colmajor_to_device(Gf, dev); torch.cuda.synchronize(); t.append(time.perf_counter())
    res = H.drive_device(Gt, J, cfg); torch.cuda.synchronize(); t.append(time.perf_counter())
    U = _device.device_to_colmajor(res.U); t.append(time.perf_counter())
    V = _device.device_to_colmajor(res.Vinv_t); t.append(time.perf_counter())
    s = res.sigma.cpu().numpy(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"as_factor {d[0]:.1f} ms, H2D {d[1]:.1f}, solve {d[2]:.1f}, U D2H {d[3]:.1f}, V D2H {d[4]:.1f}, small {d[5]:.1f}")
    t0 = time.perf_counter(); out = H.drive(G, J, cfg); print(f"drive() total {1e3*(time.perf_counter()-t0):.1f} ms")
