"""Time the GPU test-matrix pipeline (generate_factor_pair: dd generator +
dd Bunch-Parlett) at size n.  usage: python tools/bench_gen.py n [n ...]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1008_1371_b200 as H  # noqa: E402
from paper_1008_1371_b200 import factory as F  # noqa: E402

H.generate_factor_pair(H.SpectrumSpec(64, 20.0, 0))  # warm-up
for n in [int(x) for x in sys.argv[1:]]:
    spec = H.SpectrumSpec(n, 20.0, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rng = np.random.default_rng(spec.seed)
    lam = F.draw_spectrum(spec, rng)
    Mh, Ml = F._generate_dd_device(lam, rng)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    Gt, s, perm, p = F.bunch_parlett_factor_device(Mh)  # rounded-hi input: timing only
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"n": n, "generate_dd_s": t1 - t0, "bunch_parlett_s": t2 - t1}), flush=True)
