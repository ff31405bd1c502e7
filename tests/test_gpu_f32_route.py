"""Routing on the reference's own fp32 tensors (the gating layer is computed on
the fp32 hidden). Tokens here are NOT bf16-representable (make_inputs(bf16=False)), so a router that
rounded x to bf16 first would route some tokens differently (checked: the oracle's own decision on
bf16(x) differs from its decision on x at the C2 router shape). The fp32 entry points route on the
fp32 values: logits, top-K and counts are bit-exact against the oracle on the same fp32 inputs.

Tolerances as tests/test_gpu_parity.py: routing, logits, probs and combine weights bit-exact;
layer output vs the fp32 oracle rel-F <= 1e-2, max <= 3e-2 max|y| (experts take bf16(x))."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs  # noqa: E402

JOBS = os.cpu_count() or 1


def _check_decision(dec, ref, t, k):
    assert np.array_equal(dec.logits.cpu().numpy(), ref["logits"])
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), ref["topk_idx"])
    assert np.array_equal(dec.counts.cpu().numpy(), ref["counts"])
    assert dec.counts.sum().item() == t * k
    assert np.array_equal(dec.probs.cpu().numpy(), ref["probs"])
    assert np.array_equal(dec.combine_weights.cpu().numpy(), ref["combine_weights"])


# C1 router shape (router_kernel, 1 token x 4 experts), C2 router shape (router_big_kernel 4x4),
# a decode batch (router_ws_kernel) and the C3 router shape per rank (d=8192, K=4)
@pytest.mark.parametrize("t,d,n,k", [(4096, 1024, 8, 2), (16384, 4096, 16, 2), (64, 4096, 16, 2), (8192, 8192, 16, 4)])
def test_route_tokens_f32_bit_exact(t, d, n, k):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    o = Oracle("port")
    inp = make_inputs(t, d, n, 128, bf16=False, experts=False)
    ref = o.route(inp["x"], inp["w_router"], k)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=128, max_tokens=t), inp["w_router"],
                   np.zeros((n, d, 256), np.float32), np.zeros((n, 128, d), np.float32))
    dec = lay.route_tokens(torch.from_numpy(inp["x"]).cuda().contiguous())
    lay.sync()
    _check_decision(dec, ref, t, k)
    if (t, d) == (16384, 4096):
        # the fp32 entry matters: rounding x to bf16 first changes some decisions at this shape
        r16 = o.route(o.round_bf16(inp["x"]), inp["w_router"], k)
        assert not np.array_equal(r16["topk_idx"], ref["topk_idx"])
    lay.close()


def test_forward_f32_c1_shape_vs_oracle():
    """The full C1 layer (T=4096, d=1024, N=8, K=2, f=2816) on unrounded fp32 tokens: decision
    bit-exact, fp32 output within the bf16 tolerance, every row individually close (a token routed
    to another expert would be off by O(1) in its row)."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 4096, 1024, 8, 2, 2816
    o = Oracle("port")
    inp = make_inputs(t, d, n, f, bf16=False)
    ref_r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], ref_r["topk_idx"], ref_r["combine_weights"], jobs=JOBS)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), inp["w_router"], inp["w_in"],
                   inp["w_out"])
    x = torch.from_numpy(inp["x"]).cuda().contiguous()
    out, dec = lay.forward(x, want_decision=True)
    lay.sync()
    assert out.dtype == torch.float32
    _check_decision(dec, ref_r, t, k)
    o64 = out.cpu().numpy().astype(np.float64)
    d_ = o64 - ref
    assert np.linalg.norm(d_) / np.linalg.norm(ref) <= 1e-2
    assert np.abs(d_).max() <= 3e-2 * np.abs(ref).max()
    row = np.linalg.norm(d_, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    assert row.max() <= 5e-2, row.max()
    # the host-buffer fp32 entry (CL_MOE_IO_F32, the INTEGRATION.md drop-in) gives the same output
    oh = lay.forward_host(inp["x"], "f32")
    assert np.array_equal(oh, out.cpu().numpy())
    lay.close()


def test_forward_f32_decode_dense_and_sparse_agree():
    """T <= 128 takes the dense-decode path (router on a side stream): fp32 routing there too,
    bit-identical to the sparse path (CL_MOE_DENSE_DECODE is read per call)."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 64, 1024, 8, 2, 512
    o = Oracle("port")
    inp = make_inputs(t, d, n, f, bf16=False)
    ref_r = o.route(inp["x"], inp["w_router"], k)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), inp["w_router"], inp["w_in"],
                   inp["w_out"])
    x = torch.from_numpy(inp["x"]).cuda().contiguous()
    out_dense, dec = lay.forward(x, want_decision=True)
    lay.sync()
    _check_decision(dec, ref_r, t, k)
    os.environ["CL_MOE_DENSE_DECODE"] = "0"
    try:
        out_sparse = lay.forward(x)
        lay.sync()
    finally:
        del os.environ["CL_MOE_DENSE_DECODE"]
    assert torch.equal(out_dense, out_sparse)
    lay.close()
