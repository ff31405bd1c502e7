"""Time K1 and K2 inside the layer forward for the router variant forced by CL_MOE_ROUTER (read once per process).

  CL_MOE_ROUTER=ws python tools/router_timing.py 64 256 512
prints one line per T: variant, T, mean K1 (router) and K2 (plan) microseconds over 200 calls, from the
library's per-stage CUDA events (cl_moe_profile).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_09121_b200.moe import MoEConfig, MoELayer  # noqa: E402


def main(ts, d=4096, n=16, k=2, f=1024):
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=max(ts)), seed=7)
    for t in ts:
        x = lay.synthetic_tokens(t, 11)
        for _ in range(10):
            lay.forward(x)
        torch.cuda.synchronize()
        reps = 200
        lay.profile(True)
        lay.profile_read()
        for _ in range(reps):
            lay.forward(x)
        torch.cuda.synchronize()
        ms, _ = lay.profile_read()
        lay.profile(False)
        print(f"{os.environ.get('CL_MOE_ROUTER', 'auto')} T={t} router_us={ms['router'] * 1000 / reps:.1f} "
              f"plan_us={ms['plan'] * 1000 / reps:.1f}", flush=True)


if __name__ == "__main__":
    main([int(v) for v in sys.argv[1:]] or [64, 256, 512])
