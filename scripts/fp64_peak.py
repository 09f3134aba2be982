"""Measured fp64 peak of this B200 (the roofline of the multifrontal factorization kernels, a8 / a12):
cuBLAS DGEMM through torch.matmul (float64, 8192³, 2·N³ flops), best of 10 with CUDA events, plus the same
back to back for ~4 s (sustained, under the power cap).  Prints one JSON line."""
import json
import time

import torch

N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda")
b = torch.randn(N, N, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b, out=c)
    n += 1
    if n % 8 == 0:
        torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / n
fl = 2.0 * N ** 3
print(json.dumps({"fp64_dgemm_tflops": fl / (best / 1e3) / 1e12, "fp64_dgemm_tflops_sustained": fl / (sus / 1e3) / 1e12,
                  "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM), best of 10 / back to back for 4 s"}))
