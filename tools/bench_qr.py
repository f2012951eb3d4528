"""Time the GPU QR shortening (hsvd_qr_shorten) of a tall n x r factor.
usage: python tools/bench_qr.py n r"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402

n, r = int(sys.argv[1]), int(sys.argv[2])
G = np.asfortranarray(np.random.default_rng(3).standard_normal((n, r)))
H.qr_shorten(G[:64, :32].copy())  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
R, Q = H.qr_shorten(G)
t1 = time.perf_counter()
res = np.linalg.norm(Q @ R - G) / np.linalg.norm(G) if n * r <= 4096 * 2048 else None
print(json.dumps({"n": n, "r": r, "qr_s": t1 - t0, "rel_residual": res}))
