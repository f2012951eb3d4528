"""Gram timing of sweep 0 at n = 8192 (profile mode, one stream): used with
the HSVD_GRAM_NOMATH / HSVD_GRAM_NOLOAD diagnostic builds (tools/ab_variants.py)
to separate the data-movement and DMMA floors of k_gram_tma."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = np.random.default_rng(0).standard_normal((n, n))
Gt = torch.from_numpy(np.ascontiguousarray(G.T)).cuda()
J = H.SignatureVector.from_p(n, n // 2)
for _ in range(2):
    res = H.drive_device(Gt.clone(), J, H.SolverConfig(mode="block", profile=True, max_sweeps=1))
kp = res.kernel_profile
print({k: round(v["ms"], 2) for k, v in kp.items()})
