"""Where does the host-buffer path's time go at C2? Times, on one handle:
  dev      N device-resident forwards (the bench's `value` loop)
  dev+cp   the same loop while side streams copy 134 MB H2D + 134 MB D2H per call (PCIe traffic and
           its HBM / power share, without the pipeline's dependencies)
  host     N pipelined cl_moe_forward_host_async calls (the bench's `e2e` loop)
Run on the GPU box from the repo root: python tools/e2e_diag.py [N]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_09121_b200.moe import MoEConfig, MoELayer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
T, d, N, K, f = 16384, 4096, 16, 2, 14336
layer = MoELayer(MoEConfig(d_model=d, n_experts=N, top_k=K, d_ff=f, max_tokens=T, device=0), seed=20261018)
x = layer.synthetic_tokens(T, 20261018)
out = torch.empty_like(x)
st = torch.cuda.current_stream()


def fwd():
    layer._check(layer.L.cl_moe_forward(layer.h, x.data_ptr(), T, out.data_ptr(), None, st.cuda_stream), "forward")


for _ in range(5):
    fwd()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    fwd()
torch.cuda.synchronize()
dev = (time.perf_counter() - t0) / n

xh = [torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
oh = [torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
xd = [torch.empty_like(x) for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    with torch.cuda.stream(s1):
        xd[i % 2].copy_(xh[i % 2], non_blocking=True)
    with torch.cuda.stream(s2):
        oh[i % 2].copy_(xd[(i + 1) % 2], non_blocking=True)
    fwd()
torch.cuda.synchronize()
devcp = (time.perf_counter() - t0) / n

for b in xh:
    b.copy_(x)
for i in range(2):
    layer.forward_host_async(xh[i].data_ptr(), T, oh[i].data_ptr())
layer.host_wait()
t0 = time.perf_counter()
for i in range(n):
    layer.forward_host_async(xh[i % 2].data_ptr(), T, oh[i % 2].data_ptr())
layer.host_wait()
host = (time.perf_counter() - t0) / n
print(f"N={n}: dev {dev*1e3:.3f} ms   dev+copies {devcp*1e3:.3f} ms   host-buffer {host*1e3:.3f} ms per call")
layer.close()
