"""Per-sweep telemetry of a block-mode solve (rotations, skips, max|t|, ms)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
J = H.SignatureVector.from_p(n, n // 2)
Gt = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
res = H.drive_device(Gt, J, H.SolverConfig(mode="block", block_cols=32))
torch.cuda.synchronize()
for (s, rot, skip, mt), ms in zip(res.telemetry, res.sweep_gpu_ms):
    print(f"sweep {s:2d} rot {rot:10d} skip {skip:10d} frac_rot {rot/(rot+skip):.4f} max_t {mt:.3e} ms {ms:.1f}")
