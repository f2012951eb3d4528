"""One pointwise quasi-sweep at size n (for ncu captures of k_pointwise_step)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
J = H.SignatureVector.from_p(n, n // 2)
Gt = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
res = H.drive_device(Gt, J, H.SolverConfig(max_sweeps=1))
torch.cuda.synchronize()
print("sweep ms", res.sweep_gpu_ms)
