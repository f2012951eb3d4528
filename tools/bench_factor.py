"""Time the GPU Bunch-Parlett factorization (hsvd_bp_factor) at size n on a
seeded symmetric input, and the CPU oracle on a bounded sample.
usage: python tools/bench_factor.py [n] [reps] [cpu_n]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cpu_n = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rng = np.random.default_rng(0)
X = rng.standard_normal((n, n))
M = X + X.T
Mt = torch.from_numpy(M).cuda()
thresh = n * H.EPS * np.linalg.norm(M, "fro")
H.bunch_parlett_factor_device(Mt, thresh)  # warm-up
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Gt, signs, perm, p = H.bunch_parlett_factor_device(Mt, thresh)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
G = Gt.cpu().numpy().T
J = np.where(np.arange(n) < p, 1.0, -1.0)
res = np.linalg.norm((G * J) @ G.T - M) / np.linalg.norm(M) if n <= 4096 else None
# algorithmic HBM bytes of the trailing updates: the upper triangle (m^2 / 2
# elements) read and written in double-double, 16 B each way
alg_bytes = sum(16.0 * (n - k) ** 2 for k in range(1, n))
out = {"n": n, "gpu_s": min(ts), "gpu_all_s": ts, "p": p, "rel_residual": res,
       "trailing_update_GBps": alg_bytes / min(ts) / 1e9}
if cpu_n:
    sys.path.insert(0, ".")
    from oracle import oracle as O
    Xc = np.random.default_rng(0).standard_normal((cpu_n, cpu_n))
    t0 = time.perf_counter()
    O.bp_factor(Xc + Xc.T)
    tc = time.perf_counter() - t0
    out.update({"cpu_n": cpu_n, "cpu_s": tc, "cpu_extrapolated_s": tc * (n / cpu_n) ** 3,
                "cpu_note": "oracle (C, one thread, bit-exact with the reference), O(n^3) extrapolation"})
print(json.dumps(out))
