"""Measures the dense FP8 (e4m3) tensor peak of this GPU with cuBLASLt via torch._scaled_mm
(8192^3, best of 10, CUDA events) -- the FP8 denominator MEASURED_PEAKS.json does not carry.
Writes profiles/fp8_peak.json."""
import json
import os

import torch

n = 8192
a = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn)
b = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn).t()
one = torch.tensor(1.0, device="cuda")
for _ in range(3):
    torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
tf = 2 * n ** 3 / (best * 1e-3) / 1e12
out = dict(fp8_tflops=tf, how="torch._scaled_mm e4m3 8192^3 -> bf16, best of 10, CUDA events", gpu=torch.cuda.get_device_name())
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/fp8_peak.json", "w"), indent=1)
print(out)
