"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on identical inputs.

Tolerances (declared here):
  * routing indices, counts, dispatch permutation, expert offsets:   bit-exact
  * router logits:                                                    bit-exact (fp64 sequential acc)
  * probs / combine weights:                                          bit-exact (the softmax's exp is
                                                                       glibc's algorithm, csrc/glibc_exp.cuh)
  * agg_prob, aux / z loss:                                           rel 1e-6 (tile-ordered fp64 sums)
  * bf16 layer output vs fp32 oracle:   ||d||_F/||y||_F <= 1e-2 and max|d| <= 3e-2 * max|y|
  * FP8 layer output vs qdq-simulated fp32 oracle:  ||d||_F/||y||_F <= 2e-2
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs  # noqa: E402

JOBS = os.cpu_count() or 1


def _layer(inp, t, k, gemm_ctas=0, max_tokens=None):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    n, d, f2 = inp["w_in"].shape
    cfg = MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f2 // 2, max_tokens=max_tokens or t, gemm_ctas=gemm_ctas)
    return MoELayer(cfg, inp["w_router"], inp["w_in"], inp["w_out"])


def _x_dev(x):
    return torch.from_numpy(x).to("cuda").to(torch.bfloat16).contiguous()


def _rel(out, ref):
    d = out.astype(np.float64) - ref.astype(np.float64)
    rf = np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-30)
    rm = np.abs(d).max() / max(np.abs(ref).max(), 1e-30)
    return rf, rm


# T=10000 / N=16 and T=20000 / N=8 select the large-batch router variant (4 tokens x 4 experts per
# thread); the others the small-batch one.
@pytest.mark.parametrize("t,d,n,k", [(300, 256, 8, 2), (1000, 512, 16, 2), (257, 256, 16, 4), (64, 1024, 8, 1),
                                     (10000, 256, 16, 2), (20000, 256, 8, 2), (9999, 512, 32, 4)])
def test_route_tokens_bit_exact(t, d, n, k):
    o = Oracle("port")
    inp = make_inputs(t, d, n, 128, experts=False)
    inp["w_in"] = np.zeros((n, d, 256), np.float32)
    inp["w_out"] = np.zeros((n, 128, d), np.float32)
    ref = o.route(inp["x"], inp["w_router"], k)
    lay = _layer(inp, t, k)
    dec = lay.route_tokens(_x_dev(inp["x"]))
    torch.cuda.synchronize()
    lay.sync()
    assert np.array_equal(dec.logits.cpu().numpy(), ref["logits"])
    assert np.array_equal(dec.probs.cpu().numpy(), ref["probs"])
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), ref["topk_idx"])
    assert np.array_equal(dec.combine_weights.cpu().numpy(), ref["combine_weights"])
    assert np.array_equal(dec.counts.cpu().numpy(), ref["counts"])
    assert dec.counts.sum().item() == t * k
    np.testing.assert_allclose(dec.agg_prob.cpu().numpy(), ref["agg_prob"], rtol=1e-6)
    np.testing.assert_allclose(lay.aux_loss(dec), o.aux_loss(ref["probs"], ref["counts"], k), rtol=1e-6)
    np.testing.assert_allclose(lay.z_loss(dec), o.z_loss(ref["logits"]), rtol=1e-6)
    lay.close()


def test_dispatch_plan_and_copy_exact():
    o = Oracle("port")
    t, d, n, k, f = 777, 256, 8, 2, 128
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = _x_dev(inp["x"])
    out, dec = lay.forward(x, want_decision=True)
    torch.cuda.synchronize()
    idx = dec.topk_idx.cpu().numpy().astype(np.int64)
    offsets, perm, inv = o.plan(idx, n)
    assert np.array_equal(lay.stage("offsets", (n + 1,), torch.int32).cpu().numpy(), offsets)
    assert np.array_equal(lay.stage("perm", (t * k,), torch.int32).cpu().numpy(), perm)
    assert np.array_equal(lay.stage("inv", (t * k,), torch.int32).cpu().numpy(), inv)
    xp = lay.stage("x_perm", (t * k, d), torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(xp, inp["x"][perm // k])
    rw = lay.stage("row_weight", (t * k,), torch.float32).cpu().numpy()
    assert np.array_equal(rw, dec.combine_weights.cpu().numpy().ravel()[perm])
    lay.close()


@pytest.mark.parametrize("gemm_ctas", [1, 2])
def test_expert_gemms_vs_torch_fp32(gemm_ctas):
    """GEMM1 (+SwiGLU) and GEMM2 (+row weight) stage outputs against a torch fp32 reference."""
    t, d, n, k, f = 600, 512, 4, 2, 384
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k, gemm_ctas=gemm_ctas)
    out, dec = lay.forward(_x_dev(inp["x"]), want_decision=True)
    torch.cuda.synchronize()
    offsets = lay.stage("offsets", (n + 1,), torch.int32).cpu().numpy()
    xp = lay.stage("x_perm", (t * k, d), torch.bfloat16).float()
    act = lay.stage("act", (t * k, f), torch.bfloat16).float()
    y = lay.stage("y", (t * k, d), torch.bfloat16).float()
    rw = lay.stage("row_weight", (t * k,), torch.float32)
    for e in range(n):
        a, b = offsets[e], offsets[e + 1]
        if a == b:
            continue
        win = torch.from_numpy(inp["w_in"][e]).cuda()
        wout = torch.from_numpy(inp["w_out"][e]).cuda()
        h = xp[a:b] @ win
        ref_act = torch.nn.functional.silu(h[:, :f]) * h[:, f:]
        rf, rm = _rel(act[a:b].cpu().numpy(), ref_act.cpu().numpy())
        assert rf <= 1e-2 and rm <= 3e-2, (e, rf, rm)
        ref_y = (act[a:b] @ wout) * rw[a:b, None]
        rf, rm = _rel(y[a:b].cpu().numpy(), ref_y.cpu().numpy())
        assert rf <= 1e-2 and rm <= 3e-2, (e, rf, rm)
    lay.close()


@pytest.mark.parametrize("gemm_ctas", [1, 2])
@pytest.mark.parametrize("t,d,n,k,f", [(300, 256, 8, 2, 256), (1500, 512, 16, 2, 512), (129, 256, 4, 4, 128)])
def test_layer_forward_vs_oracle(gemm_ctas, t, d, n, k, f):
    o = Oracle("port")
    inp = make_inputs(t, d, n, f)
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"], jobs=JOBS)
    lay = _layer(inp, t, k, gemm_ctas=gemm_ctas)
    out = lay.forward(_x_dev(inp["x"]))
    lay.sync()
    rf, rm = _rel(out.float().cpu().numpy(), ref)
    assert rf <= 1e-2 and rm <= 3e-2, (rf, rm)
    lay.close()


@pytest.mark.slow
def test_layer_forward_c1_shape():
    """The full C1 oracle configuration (4096 tokens, d=1024, N=8, K=2, f=2816) on the GPU."""
    o = Oracle("port")
    t, d, n, k, f = 4096, 1024, 8, 2, 2816
    inp = make_inputs(t, d, n, f)
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"], jobs=JOBS)
    lay = _layer(inp, t, k)
    out, dec = lay.forward(_x_dev(inp["x"]), want_decision=True)
    lay.sync()
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), r["topk_idx"])
    rf, rm = _rel(out.float().cpu().numpy(), ref)
    assert rf <= 1e-2 and rm <= 3e-2, (rf, rm)
    lay.close()


def test_skewed_and_empty_experts_via_decision():
    """moe_forward with a caller decision: one hot expert (many m-tiles), several empty experts."""
    o = Oracle("port")
    t, d, n, k, f = 1100, 256, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    rng = np.random.default_rng(0)
    idx = np.zeros((t, k), np.int64)
    idx[:, 0] = 3
    idx[:, 1] = np.where(rng.random(t) < 0.8, 5, 0)
    w = rng.random((t, k)).astype(np.float32)
    w /= w.sum(1, keepdims=True)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], idx, w, jobs=JOBS)
    for g in (1, 2):
        lay = _layer(inp, t, k, gemm_ctas=g)
        out = lay.moe_forward(_x_dev(inp["x"]),
                              _Dec(torch.from_numpy(idx.astype(np.int32)).cuda(), torch.from_numpy(w).cuda()))
        lay.sync()
        rf, rm = _rel(out.float().cpu().numpy(), ref)
        assert rf <= 1e-2 and rm <= 3e-2, (g, rf, rm)
        lay.close()


class _Dec:
    def __init__(self, idx, w):
        self.topk_idx = idx
        self.combine_weights = w


def test_spec_moe_forward_examples():
    """K=1 -> output equals the selected expert's output exactly (weight 1);
    identical experts -> output independent of routing."""
    o = Oracle("port")
    t, d, n, f = 200, 256, 4, 128
    inp = make_inputs(t, d, n, f)
    # identical experts
    inp_same = dict(inp)
    inp_same["w_in"] = np.repeat(inp["w_in"][:1], n, 0)
    inp_same["w_out"] = np.repeat(inp["w_out"][:1], n, 0)
    lay = _layer(inp_same, t, 2)
    x = _x_dev(inp["x"])
    idx_a = np.stack([np.arange(t) % n, (np.arange(t) + 1) % n], 1).astype(np.int32)
    idx_b = np.stack([(np.arange(t) + 2) % n, (np.arange(t) + 3) % n], 1).astype(np.int32)
    w = np.full((t, 2), 0.5, np.float32)
    oa = lay.moe_forward(x, _Dec(torch.from_numpy(idx_a).cuda(), torch.from_numpy(w).cuda()))
    ob = lay.moe_forward(x, _Dec(torch.from_numpy(idx_b).cuda(), torch.from_numpy(w).cuda()))
    lay.sync()
    assert torch.equal(oa, ob)
    lay.close()
    # K=1: out == expert output (combine weight 1)
    lay = _layer(inp, t, 1)
    out, dec = lay.forward(x, want_decision=True)
    lay.sync()
    assert np.all(dec.combine_weights.cpu().numpy() == 1.0)
    e_idx = dec.topk_idx.cpu().numpy()[:, 0]
    for e in range(n):
        rows = np.where(e_idx == e)[0]
        if len(rows) == 0:
            continue
        _, y = o.expert_ffn(inp["x"][rows], inp["w_in"][e], inp["w_out"][e])
        rf, rm = _rel(out.float().cpu().numpy()[rows], y)
        assert rf <= 1e-2 and rm <= 3e-2
    lay.close()


def test_forward_host_matches_device():
    t, d, n, k, f = 333, 256, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = _x_dev(inp["x"])
    out = lay.forward(x)
    lay.sync()
    bits = x.view(torch.int16).cpu().numpy().view(np.uint16)
    out_b = lay.forward_host(bits, "bf16")
    assert np.array_equal(out_b, out.view(torch.int16).cpu().numpy().view(np.uint16))
    # pipelined host path: several calls in flight, identical results
    outs = [np.empty_like(bits) for _ in range(3)]
    for o_ in outs:
        lay.forward_host_async(bits.ctypes.data, t, o_.ctypes.data)
    lay.host_wait()
    for o_ in outs:
        assert np.array_equal(o_, out_b)
    out_f = lay.forward_host(inp["x"], "f32")
    o = Oracle("port")
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"], jobs=JOBS)
    rf, _ = _rel(out_f, ref)
    assert rf <= 1e-2
    lay.close()


def test_determinism_bitwise():
    """SPEC determinism invariant (proj/tests/tensor_test.cpp:303-314): identical inputs -> identical bits."""
    t, d, n, k, f = 512, 512, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = _x_dev(inp["x"])
    a = lay.forward(x)
    b = lay.forward(x)
    lay.sync()
    assert torch.equal(a, b)
    lay.close()


def test_errors_map_like_reference():
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer, MoEConfigError, MoEError
    inp = make_inputs(16, 256, 4, 128)
    with pytest.raises(MoEConfigError):
        MoELayer(MoEConfig(d_model=250, n_experts=4, top_k=2, d_ff=128, max_tokens=16), inp["w_router"],
                 inp["w_in"], inp["w_out"])
    with pytest.raises(MoEConfigError):
        MoELayer(MoEConfig(d_model=256, n_experts=4, top_k=5, d_ff=128, max_tokens=16), inp["w_router"],
                 inp["w_in"], inp["w_out"])
    lay = _layer(inp, 16, 2)
    x = _x_dev(inp["x"])
    with pytest.raises(MoEConfigError):
        lay.forward(torch.cat([x, x, x]).contiguous())  # exceeds max_tokens
    # non-finite hidden -> ValidationError analogue (CL_ERR_RUN) at sync
    bad = x.clone()
    bad[3, 7] = float("inf")
    lay.forward(bad)
    with pytest.raises(MoEError):
        lay.sync()
    lay.close()


def test_synthetic_weights_match_host_prng():
    """Device-side generation (cl_moe_create_synthetic) reproduces the reference Prng streams."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 256, 256, 4, 2, 128
    inp = make_inputs(t, d, n, f)
    host = _layer(inp, t, k)
    syn = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), seed=20261018)
    x = syn.synthetic_tokens(t, 20261018)
    torch.cuda.synchronize()
    xm = x.float().cpu().numpy()
    assert np.mean(xm == inp["x"]) > 0.9999
    a = host.forward(x)
    b = syn.forward(x)
    host.sync()
    syn.sync()
    assert (a == b).float().mean().item() > 0.999
    host.close()
    syn.close()


def test_device_skew_construction_matches_oracle():
    """cl_moe_synthetic_skew + shifted tokens reproduce make_inputs(skew=gamma) routing exactly."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 512, 512, 16, 2, 128
    o = Oracle("port")
    inp = make_inputs(t, d, n, f, skew=1.8)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), seed=20261018)
    lay.synthetic_skew(1.8)
    x = lay.synthetic_tokens(t, 20261018, shift=1.0)
    dec = lay.route_tokens(x)
    lay.sync()
    assert (x.float().cpu().numpy() == inp["x"]).mean() > 0.9999
    r = o.route(x.float().cpu().numpy(), inp["w_router"], k)
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), r["topk_idx"])
    assert dec.counts.cpu().numpy().max() > 0.25 * t * k  # hot expert
    lay.close()


@pytest.mark.parametrize("precision", ["bf16", "fp8"])
def test_pair_tail_tiles_match_single_cta(precision):
    """2-CTA kernels run an expert's last m-tile with <= 128 rows as an M=128 pair MMA (64 rows per
    CTA, gate/up exchanged through shared memory in the SwiGLU epilogue). The 1-CTA kernels use
    plain M=128 tiles; both accumulate every output element in the same K order, so the layer
    outputs must agree bit for bit. Many experts give tail sizes across 1..255."""
    t, d, n, k, f = 12000, 256, 64, 4, 256
    inp = make_inputs(t, d, n, f)
    x = _x_dev(inp["x"])
    outs = []
    for g in (1, 2):
        lay = _layer(inp, t, k, gemm_ctas=g)
        if precision == "fp8":
            lay.calibrate(x)
            lay.quantize_fp8()
        outs.append(lay.forward(x))
        lay.sync()
    counts = Oracle("port").route(inp["x"], inp["w_router"], k)["counts"]
    tails = counts % 256
    assert ((tails > 0) & (tails <= 128)).sum() >= 10 and (tails > 128).sum() >= 5
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("gemm_ctas", [1, 2])
@pytest.mark.parametrize("t,d,n,k,f", [(1, 256, 128, 8, 128), (7, 256, 1, 1, 128), (5, 512, 128, 1, 256),
                                       (64, 8192, 4, 2, 128), (1000, 256, 64, 8, 128), (2, 256, 2, 2, 384)])
def test_layer_forward_edge_shapes(gemm_ctas, t, d, n, k, f):
    """Limits of the configuration space: one token, one expert, N = 128 with K = 8 (most experts
    empty), the widest hidden size at a tiny batch, f not a multiple of 256."""
    o = Oracle("port")
    inp = make_inputs(t, d, n, f)
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"], jobs=JOBS)
    lay = _layer(inp, t, k, gemm_ctas=gemm_ctas)
    out, dec = lay.forward(_x_dev(inp["x"]), want_decision=True)
    lay.sync()
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), r["topk_idx"])
    assert np.array_equal(dec.counts.cpu().numpy(), r["counts"])
    rf, rm = _rel(out.float().cpu().numpy(), ref)
    assert rf <= 1e-2 and rm <= 3e-2, (rf, rm)
    lay.close()


def test_forward_graph_replays_bit_identically():
    """cl_moe_forward_graph: captured once per (buffers, T, precision), replayed after."""
    t, d, n, k, f = 200, 512, 16, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = _x_dev(inp["x"])
    ref = lay.forward(x)
    out = torch.empty_like(x)
    for _ in range(3):
        out.zero_()
        lay.forward_graph(x, out)
        lay.sync()
        assert torch.equal(out, ref)
    xs = x[:77].contiguous()  # a different T -> a second graph
    o2 = lay.forward_graph(xs)
    assert torch.equal(o2, lay.forward(xs))
    lay.calibrate(x)
    lay.quantize_fp8()  # precision is part of the key
    ref8 = lay.forward(x)
    lay.forward_graph(x, out)
    lay.sync()
    assert torch.equal(out, ref8)
