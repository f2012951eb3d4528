"""Per-kernel device time of one chosen sweep of the n=8192 block solve
(profile mode: one stream, no graph; HSVD_PROFILE_SWEEP picks the sweep).
usage: HSVD_PROFILE_SWEEP=k python tools/profile_sweep.py [n]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = np.random.default_rng(0).standard_normal((n, n))
Gt = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
J = H.SignatureVector.from_p(n, n // 2)
res = H.drive_device(Gt.clone(), J, H.SolverConfig(mode="block", profile=True))
print("sweeps", res.sweeps_used, "kernel profile", res.kernel_profile)
print("sweep ms", [round(x, 1) for x in res.sweep_gpu_ms])
