"""Where does the time of one drive_device call go?  (wall, events, phases)"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
order = sys.argv[2] if len(sys.argv) > 2 else "oriented"
G = np.random.default_rng(0).standard_normal((n, n))
J = H.SignatureVector.from_p(n, n // 2)
G0 = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
Gw = torch.empty_like(G0)
cfg = H.SolverConfig(mode="block", block_cols=32, inner_ordering=order)
s = torch.cuda.current_stream()
for it in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    Gw.copy_(G0)
    t1 = time.perf_counter()
    res = H.drive_device(Gw, J, cfg)
    t2 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"it {it}: events {e0.elapsed_time(e1):.1f} ms, wall {1e3*(t3-t0):.1f} "
          f"(copy enqueue {1e3*(t1-t0):.1f}, drive {1e3*(t2-t1):.1f}), phases {res.host_phase_ms}, "
          f"sum sweeps {sum(res.sweep_gpu_ms):.1f}, sweeps {res.sweeps_used}", flush=True)
