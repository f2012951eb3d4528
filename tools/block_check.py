"""Print block-mode accuracy/sweeps/time against the oracle for a few sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.block_metrics import residuals, sigma_class_reldiff  # noqa: E402
from tests.golden.inputs import make_case_input  # noqa: E402

for (n, p, kind, b) in [(256, 128, "gauss", 16), (256, 128, "gauss", 32), (512, 384, "gauss", 32),
                        (1024, 512, "gauss", 32), (1024, 1024, "gauss", 32),
                        (2048, 1024, "graded10", 32)]:
    G = make_case_input(n, n, 0, kind)
    signs = np.array([1] * p + [-1] * (n - p), np.int8)
    t = time.time()
    ref = O.drive(G, signs, p, workers=16)
    tr = time.time() - t
    for inner in ("oriented", "full"):
        cfg = H.SolverConfig(mode="block", block_cols=b, inner_ordering=inner)
        H.drive(G, H.SignatureVector(signs, p), cfg)
        torch.cuda.synchronize()
        t = time.time()
        res = H.drive(G, H.SignatureVector(signs, p), cfg)
        tg = time.time() - t
        d = sigma_class_reldiff(res.sigma, res.lam, ref.sigma, ref.lam)
        rb, rr = residuals(G, res, signs), residuals(G, ref, signs)
        print(f"n={n} p={p} {kind} b={b} {inner}: sweeps {res.sweeps_used} (ref {ref.sweeps_used}) "
              f"{res.stop_reason} sigma_rel {d:.2e} | dU {rb['dU']:.2e} ({rb['dU']/rr['dU']:.2f}x) "
              f"vjv {rb['vjv']:.2e} ({rb['vjv']/rr['vjv']:.2f}x) recon {rb['recon']:.2e} "
              f"({rb['recon']/rr['recon']:.2f}x) | gpu {tg:.3f}s cpu-oracle {tr:.2f}s "
              f"sweep_ms {[round(x,2) for x in res.sweep_gpu_ms[:3]]}", flush=True)
