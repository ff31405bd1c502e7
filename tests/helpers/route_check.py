"""Subprocess helper for tests/test_gpu_router_variants.py: route one batch on the GPU with the
router variant forced by CL_MOE_ROUTER (read once per process) and compare with the oracle."""
import sys

import numpy as np
import torch

from oracle.oracle import Oracle, make_inputs, router_fp8_sim
from paper_2509_09121_b200.moe import MoEConfig, MoELayer


def main(t, d, n, k, mode="random", dtype="bf16"):
    # dtype "f32": unrounded fp32 tokens routed through the fp32 entry (cl_moe_route_tokens_f32);
    # "fp8": bf16 tokens through the router of the FP8 scheme (qdq'd x and W_r)
    f32 = dtype == "f32"
    inp = make_inputs(t, d, n, 128, experts=False, bf16=not f32)
    if mode == "ties":
        # exact ties: odd router columns duplicate the even ones (equal logits -> equal probs, the
        # lowest index must win), every 7th token is all-zero (uniform probs -> experts 0..K-1),
        # and the last expert's column is zero
        wr = inp["w_router"]
        wr[:, 1::2] = wr[:, 0:(n // 2) * 2:2]
        wr[:, n - 1] = 0.0
        inp["x"][::7] = 0.0
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=128, max_tokens=t), inp["w_router"],
                   np.zeros((n, d, 256), np.float32), np.zeros((n, 128, d), np.float32))
    xd = torch.from_numpy(inp["x"]).cuda()
    if dtype == "fp8":
        # the router under the FP8 scheme: E4M3 codes of x / s_x into K1
        s_r = float(np.float32(np.abs(inp["x"]).max()) / np.float32(448))
        lay.quantize_fp8(np.ones(n, np.float32), np.ones(n, np.float32), router_act_scale=s_r)
        ref, _ = router_fp8_sim(Oracle("port"), inp["x"], inp["w_router"], k, s_r)
    dec = lay.route_tokens(xd.contiguous() if f32 else xd.to(torch.bfloat16))
    lay.sync()
    if dtype != "fp8":
        ref = Oracle("port").route(inp["x"], inp["w_router"], k)
    ok = (np.array_equal(dec.logits.cpu().numpy(), ref["logits"]) and
          np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), ref["topk_idx"]) and
          np.array_equal(dec.counts.cpu().numpy(), ref["counts"]) and
          np.array_equal(dec.probs.cpu().numpy(), ref["probs"]) and
          np.array_equal(dec.combine_weights.cpu().numpy(), ref["combine_weights"]))
    print("ok" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(*map(int, sys.argv[1:5]), *sys.argv[5:7]))
