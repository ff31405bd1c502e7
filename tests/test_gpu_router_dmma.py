"""The fp64 tensor-core router (router_dmma_kernel, DESIGN.md §4 K1): mma.sync.m8n8k4.f64 evaluates
its four k-steps as the sequential FMA chain, so one DMMA is four steps of the reference's
ascending-l logit chain (tensor.cpp:157-173). The handle checks the instruction on the device at
creation; on the B200 the check passes and batches beyond the decode sizes take this kernel.
Decisions (logits, probs, top-K, combine weights, counts) are bit-exact against the oracle, for
bf16 and fp32 input, at the C1 and C2 router shapes; decode-size batches keep the warp-specialised
chain kernel. (tests/test_gpu_router_variants.py forces the variant over the whole shape sweep.)"""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle, make_inputs

pytestmark = pytest.mark.gpu


def _layer(inp, t, k):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    n, d, f2 = inp["w_in"].shape
    return MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f2 // 2, max_tokens=t), inp["w_router"],
                    inp["w_in"], inp["w_out"])


@pytest.mark.parametrize("t,d,n,k,bf16", [(4096, 1024, 8, 2, True), (16384, 4096, 16, 2, True),
                                          (16384, 4096, 16, 2, False), (9000, 512, 32, 4, True),
                                          (5000, 256, 4, 1, False), (7000, 512, 12, 3, True)])
def test_dmma_router_bit_exact(t, d, n, k, bf16):
    o = Oracle("port")
    inp = make_inputs(t, d, n, 128, experts=False, bf16=bf16)
    inp["w_in"] = np.zeros((n, d, 256), np.float32)
    inp["w_out"] = np.zeros((n, 128, d), np.float32)
    ref = o.route(inp["x"], inp["w_router"], k)
    lay = _layer(inp, t, k)
    x = torch.from_numpy(inp["x"]).cuda()
    dec = lay.route_tokens(x.to(torch.bfloat16) if bf16 else x.contiguous())
    lay.sync()
    variant, ok = lay.router_variant()
    assert ok, "the DMMA device check failed on this GPU"
    assert variant == 5, variant
    assert np.array_equal(dec.logits.cpu().numpy(), ref["logits"])
    assert np.array_equal(dec.probs.cpu().numpy(), ref["probs"])
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), ref["topk_idx"])
    assert np.array_equal(dec.combine_weights.cpu().numpy(), ref["combine_weights"])
    assert np.array_equal(dec.counts.cpu().numpy(), ref["counts"])
    lay.close()


def test_expert_counts_beyond_the_dmma_tiles_fall_back():
    """N = 20 (three 8-expert tiles: not instantiated) routes with the DFMA kernels, still exact."""
    t, d, n, k = 6000, 256, 20, 2
    o = Oracle("port")
    inp = make_inputs(t, d, n, 128, experts=False)
    inp["w_in"] = np.zeros((n, d, 256), np.float32)
    inp["w_out"] = np.zeros((n, 128, d), np.float32)
    ref = o.route(inp["x"], inp["w_router"], k)
    lay = _layer(inp, t, k)
    dec = lay.route_tokens(torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16))
    lay.sync()
    assert lay.router_variant()[0] != 5
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), ref["topk_idx"])
    assert np.array_equal(dec.probs.cpu().numpy(), ref["probs"])
    lay.close()


def test_decode_batches_keep_the_chain_kernel():
    inp = make_inputs(64, 1024, 16, 128, experts=False)
    inp["w_in"] = np.zeros((16, 1024, 256), np.float32)
    inp["w_out"] = np.zeros((16, 128, 1024), np.float32)
    lay = _layer(inp, 64, 2)
    lay.route_tokens(torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16))
    lay.sync()
    assert lay.router_variant()[0] == 4
    lay.close()
