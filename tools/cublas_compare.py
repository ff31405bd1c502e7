"""Same-box comparison: cuBLAS (torch.bmm, bf16) on the balanced C2 expert shapes vs this
repo's grouped GEMMs (stage times from bench.py). Timed back to back for ~3 s each (sustained,
power-capped), CUDA events."""
import json
import sys
import time

import torch

E, M, D, F = 16, 2048, 4096, 14336


def timeit(fn, secs=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n, t0 = 0, time.time()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < secs:
        fn()
        n += 1
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


x = torch.randn(E, M, D, device="cuda", dtype=torch.bfloat16)
w1 = torch.randn(E, D, 2 * F, device="cuda", dtype=torch.bfloat16)
a = torch.randn(E, M, F, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(E, F, D, device="cuda", dtype=torch.bfloat16)
g1 = timeit(lambda: torch.bmm(x, w1))
g2 = timeit(lambda: torch.bmm(a, w2))
f1 = 2 * E * M * D * 2 * F
f2 = 2 * E * M * F * D
out = dict(cublas_gemm1_ms=g1, cublas_gemm1_tflops=f1 / g1 / 1e9, cublas_gemm2_ms=g2, cublas_gemm2_tflops=f2 / g2 / 1e9,
           note="torch.bmm bf16 (no SwiGLU / no row scale), sustained ~3 s loops")
print(json.dumps(out))
