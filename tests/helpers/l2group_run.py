"""Subprocess helper for tests/test_gpu_l2_group.py: one layer run (bf16 forward, FP8 forward,
training step) whose outputs are saved to an .npz; CL_MOE_L2_GROUP_MB (read once per process)
sets the L2 tile-group budget of the grouped GEMMs (m-tile groups of GEMM1/GEMM2, the weight-
gradient GEMMs' group bytes)."""
import sys

import numpy as np
import torch

from oracle.oracle import make_inputs
from paper_2509_09121_b200.moe import MoEConfig, MoELayer


def main(path, t, d, n, k, f):
    inp = make_inputs(t, d, n, f)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), inp["w_router"], inp["w_in"],
                   inp["w_out"])
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    g = torch.from_numpy(make_inputs(t, d, 1, f, seed=77, experts=False)["x"]).cuda().to(torch.bfloat16).contiguous()
    res = {}
    res["out_bf16"] = lay.forward(x)
    lay.forward_train(x)
    dh, dcw, dwi, dwo = lay.backward(g)
    res.update(d_hidden=dh, d_combine_w=dcw, dw_in=dwi, dw_out=dwo)
    lay.calibrate(x)
    lay.quantize_fp8()
    res["out_fp8"] = lay.forward(x)
    lay.sync()
    np.savez(path, **{k_: (v.view(torch.int16) if v.dtype == torch.bfloat16 else v).cpu().numpy()
                      for k_, v in res.items()})
    print("ok")


if __name__ == "__main__":
    main(sys.argv[1], *map(int, sys.argv[2:7]))
