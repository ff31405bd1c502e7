"""The certified large-batch router of the fused forward (csrc/router_cert.cuh, opt-in via
CL_MOE_ROUTER_CERT=1): fp32 logits with a
rigorous error bound decide the tokens whose top-K order is unambiguous, the rest are recomputed
with the reference's exact fp64 chains. What the fused forward consumes — routing indices, counts,
expert offsets and the dispatch permutation — must be bit-exact against the oracle (checked through
the stage buffers of a forward WITHOUT a decision export, i.e. the certified path), including exact
and near ties, which must fall back to the exact chains; the layer output stays within the bf16
tolerance of the oracle and within ~1e-3 of the exact-router forward (combine weights of certified
tokens come from the fp32 logits)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs, router_fp8_sim  # noqa: E402

JOBS = os.cpu_count() or 1


@pytest.fixture(autouse=True)
def _cert_on():
    """The certified router is opt-in (CL_MOE_ROUTER_CERT=1, read per call)."""
    old = os.environ.get("CL_MOE_ROUTER_CERT")
    os.environ["CL_MOE_ROUTER_CERT"] = "1"
    yield
    if old is None:
        del os.environ["CL_MOE_ROUTER_CERT"]
    else:
        os.environ["CL_MOE_ROUTER_CERT"] = old


def _layer(inp, t, k):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    n, d, f2 = inp["w_in"].shape
    return MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f2 // 2, max_tokens=t), inp["w_router"],
                    inp["w_in"], inp["w_out"])


def _plan_check(lay, ref_idx, n, t, k):
    o = Oracle("port")
    offsets, perm, inv = o.plan(ref_idx, n)
    assert np.array_equal(lay.stage("offsets", (n + 1,), torch.int32).cpu().numpy(), offsets)
    assert np.array_equal(lay.stage("perm", (t * k,), torch.int32).cpu().numpy(), perm)
    assert np.array_equal(lay.stage("inv", (t * k,), torch.int32).cpu().numpy(), inv)


def _certified_forward(lay, x):
    calls0, _ = lay.router_stats()
    out = lay.forward(x)
    lay.sync()
    calls1, recomputed = lay.router_stats()
    assert calls1 == calls0 + 1, "the fused forward did not take the certified router"
    return out, recomputed


@pytest.mark.parametrize("t,d,n,k,f,mode", [
    (16384, 512, 16, 2, 256, "random"), (10000, 1024, 8, 1, 256, "random"), (8192, 256, 32, 4, 256, "random"),
    (6000, 4096, 16, 2, 256, "random"), (9000, 512, 16, 2, 256, "ties"), (9000, 512, 16, 4, 256, "near"),
    (12000, 512, 12, 3, 256, "random")])
def test_certified_routing_bit_exact(t, d, n, k, f, mode):
    o = Oracle("port")
    inp = make_inputs(t, d, n, f)
    if mode == "ties":  # duplicated router columns (equal logits) and all-zero tokens (uniform probs)
        inp["w_router"][:, 1::2] = inp["w_router"][:, 0:(n // 2) * 2:2]
        inp["x"][::5] = 0.0
    elif mode == "near":  # logits a few fp64 ulps apart: only the exact chains can order them
        inp["w_router"][:, 3] = inp["w_router"][:, 2] * np.float32(1.0 + 2.0 ** -23)
        inp["w_router"][:, 5] = np.nextafter(inp["w_router"][:, 4], np.float32(np.inf))
    r = o.route(inp["x"], inp["w_router"], k)
    lay = _layer(inp, t, k)
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    out, recomputed = _certified_forward(lay, x)
    _plan_check(lay, r["topk_idx"], n, t, k)
    if mode == "random":
        assert recomputed < 0.05 * t, recomputed
    else:
        assert recomputed > 0  # the ties / near-ties must have been sent to the exact chains
    exact, dec = lay.forward(x, want_decision=True)  # decision export: the exact router
    lay.sync()
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), r["topk_idx"])
    a, b = out.float().cpu().numpy(), exact.float().cpu().numpy()
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-3
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"], jobs=JOBS)
    assert np.linalg.norm(a - ref) / np.linalg.norm(ref) <= 1e-2
    print(f"T={t} N={n} K={k} {mode}: {recomputed} tokens recomputed exactly")
    lay.close()


def test_certified_routing_fp32_input_and_fp8_router():
    """fp32 hidden (routed on its own values) and the FP8 scheme's router (E4M3 codes): the
    certified path's permutation equals the oracle's for each."""
    t, d, n, k, f = 12000, 1024, 16, 2, 256
    o = Oracle("port")
    inp = make_inputs(t, d, n, f, bf16=False)
    lay = _layer(inp, t, k)
    x32 = torch.from_numpy(inp["x"]).cuda().contiguous()
    _certified_forward(lay, x32)
    _plan_check(lay, o.route(inp["x"], inp["w_router"], k)["topk_idx"], n, t, k)
    xb = x32.to(torch.bfloat16).contiguous()
    lay.calibrate(xb)
    lay.quantize_fp8()
    _, recomputed = _certified_forward(lay, xb)
    s_r = lay.router_fp8_scales()[1]
    rq, _ = router_fp8_sim(o, xb.float().cpu().numpy(), lay.router_weights(), k, s_r)
    _plan_check(lay, rq["topk_idx"], n, t, k)
    assert recomputed < 0.05 * t
    lay.close()


def test_certified_routing_off_by_default():
    """Without CL_MOE_ROUTER_CERT=1 every call takes the exact kernels."""
    inp = make_inputs(8000, 256, 16, 128)
    lay = _layer(inp, 8000, 2)
    del os.environ["CL_MOE_ROUTER_CERT"]
    lay.forward(torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous())
    lay.sync()
    assert lay.router_stats()[0] == 0
    os.environ["CL_MOE_ROUTER_CERT"] = "1"
    lay.close()
