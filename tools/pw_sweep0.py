"""Time pointwise sweep 0 at size n (device-resident, one sweep)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
J = H.SignatureVector.from_p(n, n // 2)
Gt0 = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
for it in range(2):
    Gt = Gt0.clone()
    res = H.drive_device(Gt, J, H.SolverConfig(max_sweeps=2))
    torch.cuda.synchronize()
    print(f"n={n} pointwise sweeps 0-1 ms {[round(x, 1) for x in res.sweep_gpu_ms]}, rot {res.rotations}")
