"""Measure the FP64 roofline denominator on this B200: cuBLAS DGEMM
(torch.matmul float64) n^3, best of 10 after warm-up, CUDA events."""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    c = a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
tf = 2 * n ** 3 / (best / 1e3) / 1e12
print(json.dumps({"dgemm_n": n, "best_ms": best, "fp64_tflops": tf}))
