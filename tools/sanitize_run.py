"""Small invocations of the hot-path kernels for compute-sanitizer (tools/sanitize.sh): the router
variants (CL_MOE_ROUTER picks one per process), plan, dispatch, both grouped-GEMM instantiations
(cta_group::1 / ::2; bf16 and FP8), combine, dense decode and one training step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import make_inputs  # noqa: E402
from paper_2509_09121_b200.moe import MoEConfig, MoELayer  # noqa: E402


def main(what):
    t, d, n, k, f = 300, 256, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    for g in (1, 2):
        lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t, gemm_ctas=g),
                       inp["w_router"], inp["w_in"], inp["w_out"])
        lay.forward(x)
        if what == "all":
            lay.forward(x[:64].contiguous())  # dense decode
            lay.forward_train(x)
            lay.backward_full(x, 0.01, 0.001)
            lay.calibrate(x)
            lay.quantize_fp8()
            lay.forward(x)
        lay.sync()
        lay.close()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
