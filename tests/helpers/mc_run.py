"""Subprocess helper for tests/test_gpu_gemm_multicast.py: bf16 and FP8 forwards of one layer,
outputs saved to an .npz; CL_MOE_GEMM_MC (read once per process) selects the clusters of two CTA
pairs sharing the B tile by TMA multicast."""
import sys

import numpy as np
import torch

from oracle.oracle import make_inputs
from paper_2509_09121_b200.moe import MoEConfig, MoELayer


def main(path, t, d, n, k, f):
    inp = make_inputs(t, d, n, f)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t, gemm_ctas=2), inp["w_router"],
                   inp["w_in"], inp["w_out"])
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    res = {"bf16": lay.forward(x)}
    res["act_bf16"] = lay.stage("act", (t * k, f), torch.bfloat16)
    lay.calibrate(x)
    lay.quantize_fp8()
    res["fp8"] = lay.forward(x)
    lay.sync()
    np.savez(path, **{k_: v.view(torch.int16).cpu().numpy() for k_, v in res.items()})
    print("ok")


if __name__ == "__main__":
    main(sys.argv[1], *map(int, sys.argv[2:7]))
