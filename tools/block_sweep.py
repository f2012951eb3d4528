"""One (or a few) block-mode quasi-sweeps at size n, for ncu captures of the
block kernels.  usage: python tools/block_sweep.py [n] [max_sweeps] [b] [ordering] [streams]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
b = int(sys.argv[3]) if len(sys.argv) > 3 else 32
order = sys.argv[4] if len(sys.argv) > 4 else "full"
streams = int(sys.argv[5]) if len(sys.argv) > 5 else 2
G = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
J = H.SignatureVector.from_p(n, n // 2)
Gt = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
res = H.drive_device(Gt, J, H.SolverConfig(mode="block", block_cols=b, max_sweeps=sweeps,
                                           use_graph=False, inner_ordering=order,
                                           block_streams=streams))
torch.cuda.synchronize()
print("sweep ms", res.sweep_gpu_ms)
