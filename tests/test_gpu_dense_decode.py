"""Dense decode (host_forward.cuh run_forward): at T <= 128 every expert runs all tokens and the
router runs beside GEMM1 on a side stream. Outputs and the routing decision must be bit-identical
to the sparse path (CL_MOE_DENSE_DECODE=0), for bf16 and FP8, through the device, graph and
host-buffer entry points; and bf16 outputs stay within the declared tolerance of the oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs  # noqa: E402


def _layer(inp, t, k, max_tokens=None):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    n, d, f2 = inp["w_in"].shape
    return MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f2 // 2, max_tokens=max_tokens or t),
                    inp["w_router"], inp["w_in"], inp["w_out"])


def _run(lay, x, dense, entry="device"):
    os.environ["CL_MOE_DENSE_DECODE"] = "1" if dense else "0"
    try:
        if entry == "graph":
            out = lay.forward_graph(x)
            lay.sync()
            return out.cpu().clone(), None
        if entry == "host":  # bf16 bits in and out of host buffers
            out = lay.forward_host(x.cpu().view(torch.int16).numpy().view(np.uint16))
            return torch.from_numpy(out.view(np.int16)).view(torch.bfloat16).clone(), None
        out, dec = lay.forward(x, want_decision=True)
        lay.sync()
        return out.cpu().clone(), (dec.topk_idx.cpu().clone(), dec.combine_weights.cpu().clone(),
                                   dec.counts.cpu().clone(), dec.probs.cpu().clone())
    finally:
        os.environ.pop("CL_MOE_DENSE_DECODE", None)


@pytest.mark.parametrize("t,d,n,k,f", [(1, 256, 8, 2, 128), (5, 256, 16, 2, 256), (64, 512, 16, 2, 256),
                                       (128, 256, 4, 1, 128), (37, 256, 128, 8, 128), (100, 512, 32, 4, 384),
                                       (3, 256, 1, 1, 128)])
def test_dense_decode_bit_identical_to_sparse(t, d, n, k, f):
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    ys, ds = _run(lay, x, dense=False)
    yd, dd = _run(lay, x, dense=True)
    assert torch.equal(ys.view(torch.int16), yd.view(torch.int16))
    for a, b in zip(ds, dd):
        assert torch.equal(a, b)
    # and the dense path itself against the oracle (bf16 tolerance)
    o = Oracle("port")
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"])
    dy = yd.float().numpy().astype(np.float64) - ref
    assert np.linalg.norm(dy) / np.linalg.norm(ref) <= 1e-2
    lay.close()


@pytest.mark.parametrize("entry", ["graph", "host"])
def test_dense_decode_entry_points(entry):
    t, d, n, k, f = 48, 256, 16, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    ys, _ = _run(lay, x, dense=False)
    yd, _ = _run(lay, x, dense=True, entry=entry)
    assert torch.equal(ys.view(torch.int16), yd.to(torch.bfloat16).view(torch.int16))
    lay.close()


@pytest.mark.parametrize("t", [1, 64, 128])
def test_dense_decode_fp8_bit_identical_to_sparse(t):
    d, n, k, f = 512, 8, 2, 256
    inp = make_inputs(max(t, 256), d, n, f)
    lay = _layer(inp, max(t, 256), k)
    xc = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    lay.calibrate(xc)
    lay.quantize_fp8()
    x = xc[:t].contiguous()
    ys, ds = _run(lay, x, dense=False)
    yd, dd = _run(lay, x, dense=True)
    assert torch.equal(ys.view(torch.int16), yd.view(torch.int16))
    for a, b in zip(ds, dd):
        assert torch.equal(a, b)
    lay.close()


def test_dense_decode_stage_profile():
    """Per-stage timing events of the dense path (router/plan on the side stream) read back sanely."""
    t, d, n, k, f = 64, 256, 16, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    lay.forward(x)
    lay.sync()
    lay.profile(True)
    for _ in range(3):
        lay.forward(x)
    lay.sync()
    ms, calls = lay.profile_read()
    lay.profile(False)
    assert calls[0] == 3
    for name in ("router", "dispatch", "gemm1", "gemm2", "combine"):
        assert ms[name] > 0.0, (name, ms)
    assert ms["plan"] >= 0.0  # the plan runs inside the router's last CTA here: may read ~0
    lay.close()


def test_dense_decode_stage_view():
    """After a dense-decode forward the stage buffers are the dense ones (rows = N*T, row e*T + t =
    token t for expert e), not stale buffers of an earlier sparse call; perm is not materialised."""
    from paper_2509_09121_b200.moe import MoEError
    t, d, n, k, f = 64, 256, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = _layer(inp, t, k)
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    os.environ["CL_MOE_DENSE_DECODE"] = "0"
    try:
        lay.forward(x)  # a sparse call first: its buffers must not leak into the dense view
        lay.sync()
        ys = lay.stage("y", (t * k, d), torch.bfloat16).clone()
        inv_s = lay.stage("inv", (t * k,), torch.int32).clone()
    finally:
        del os.environ["CL_MOE_DENSE_DECODE"]
    _, dec = lay.forward(x, want_decision=True)
    lay.sync()
    idx = dec.topk_idx.cpu().numpy()
    w = dec.combine_weights.cpu().numpy()
    assert np.array_equal(lay.stage("offsets", (n + 1,), torch.int32).cpu().numpy(), np.arange(n + 1) * t)
    inv = lay.stage("inv", (t * k,), torch.int32).cpu().numpy().reshape(t, k)
    assert np.array_equal(inv, idx * t + np.arange(t)[:, None])
    rw = lay.stage("row_weight", (n * t,), torch.float32).cpu().numpy().reshape(n, t)
    want = np.zeros((n, t), np.float32)
    for j in range(t):
        for kk in range(k):
            want[idx[j, kk], j] = w[j, kk]
    assert np.array_equal(rw, want)
    # the routed dense rows carry exactly the sparse path's weighted expert outputs
    yd = lay.stage("y", (n * t, d), torch.bfloat16)
    assert torch.equal(yd[torch.from_numpy(inv.reshape(-1)).long().cuda()], ys[inv_s.long()])
    with pytest.raises(MoEError, match="perm"):
        lay.stage("perm", (t * k,), torch.int32)
    lay.close()
