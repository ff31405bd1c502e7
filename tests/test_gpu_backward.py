"""GPU expert-FFN backward vs the oracle's layer backward (the reference Tape, restated and pinned
bit-exact against oracle/_ref in tests/test_oracle.py).

Tolerances (bf16 operands and intermediates vs the fp32 oracle on the same bf16-valued inputs):
d_hidden, dW_in, dW_out: ||d||_F/||ref||_F <= 2e-2; d_combine_w: <= 2e-2. Experts with no routed
token must get exactly zero weight gradients."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs  # noqa: E402

JOBS = os.cpu_count() or 1


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("gemm_ctas", [1, 2])
@pytest.mark.parametrize("t,d,n,k,f", [(300, 256, 4, 2, 256), (1100, 512, 8, 2, 512), (37, 256, 8, 1, 256),
                                       (1, 256, 8, 2, 256), (20, 256, 64, 2, 256), (9, 256, 128, 8, 256)])
def test_backward_vs_oracle(gemm_ctas, t, d, n, k, f):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    o = Oracle("port")
    inp = make_inputs(t, d, n, f)
    g = make_inputs(t, d, 1, f, seed=77, experts=False)["x"]  # bf16-valued dOut
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t, gemm_ctas=gemm_ctas),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    out, dec = lay.forward_train(x, want_decision=True)
    dh, dcw, dwi, dwo = lay.backward(torch.from_numpy(g).cuda().to(torch.bfloat16).contiguous())
    lay.sync()
    idx = dec.topk_idx.cpu().numpy().astype(np.int64)
    w = dec.combine_weights.cpu().numpy()
    r = o.route(inp["x"], inp["w_router"], k)
    assert np.array_equal(idx, r["topk_idx"])
    ref_out = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], idx, w, jobs=JOBS)
    assert _rel(out.float().cpu().numpy(), ref_out) <= 1e-2
    rdh, rdcw, rdwi, rdwo = o.moe_backward(inp["x"], inp["w_in"], inp["w_out"], idx, w, g, jobs=JOBS)
    assert _rel(dh.float().cpu().numpy(), rdh) <= 2e-2
    assert _rel(dcw.cpu().numpy(), rdcw) <= 2e-2
    gwi, gwo = dwi.cpu().numpy(), dwo.cpu().numpy()
    counts = np.bincount(idx.ravel(), minlength=n)
    for e in range(n):
        if counts[e] == 0:
            assert not gwi[e].any() and not gwo[e].any()
        else:
            assert _rel(gwi[e], rdwi[e]) <= 2e-2, (e, _rel(gwi[e], rdwi[e]))
            assert _rel(gwo[e], rdwo[e]) <= 2e-2, (e, _rel(gwo[e], rdwo[e]))
    lay.close()


def test_backward_requires_forward_train():
    from paper_2509_09121_b200.moe import MoEConfig, MoEConfigError, MoELayer
    inp = make_inputs(16, 256, 4, 256)
    lay = MoELayer(MoEConfig(d_model=256, n_experts=4, top_k=2, d_ff=256, max_tokens=16), inp["w_router"],
                   inp["w_in"], inp["w_out"])
    with pytest.raises(MoEConfigError):
        lay.backward(torch.zeros(16, 256, dtype=torch.bfloat16, device="cuda"))
    lay.close()


@pytest.mark.parametrize("t,d,n,k,f,ga,gz", [(300, 256, 8, 2, 256, 0.01, 0.001), (257, 512, 16, 4, 256, 1.0, 1.0),
                                             (2000, 256, 16, 1, 256, 0.1, 0.0)])
def test_full_backward_with_router_vs_oracle(t, d, n, k, f, ga, gz):
    """Layer + router backward (aux / Z loss weighted by g_aux / g_z) vs the oracle, which is
    itself pinned against the reference Tape in tests/test_oracle.py."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    o = Oracle("port")
    inp = make_inputs(t, d, n, f)
    g = make_inputs(t, d, 1, f, seed=77, experts=False)["x"]
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    lay.forward_train(x)
    dh, dwr, dwi, dwo = lay.backward_full(torch.from_numpy(g).cuda().to(torch.bfloat16).contiguous(), ga, gz)
    lay.sync()
    rdh, rdwr, rdwi, rdwo = o.moe_backward_full(inp["x"], inp["w_router"], inp["w_in"], inp["w_out"], g, ga, gz, k,
                                                jobs=JOBS)
    assert _rel(dh.float().cpu().numpy(), rdh) <= 2e-2
    assert _rel(dwr.cpu().numpy(), rdwr) <= 2e-2, _rel(dwr.cpu().numpy(), rdwr)
    assert _rel(dwi.cpu().numpy(), rdwi) <= 2e-2
    assert _rel(dwo.cpu().numpy(), rdwo) <= 2e-2
    lay.close()


def test_training_forward_keeps_dispatched_rows_padded():
    """A single-GPU forward_train writes the dispatched rows and the SwiGLU output only into the
    padded layouts the weight gradients (and GEMM1 / GEMM2) read: the x_perm and act stages are
    then refused (stage contract, compass_moe.h), and an inference forward afterwards materialises
    them again."""
    from paper_2509_09121_b200.moe import MoEConfig, MoEError, MoELayer
    t, d, n, k, f = 300, 256, 4, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), inp["w_router"],
                   inp["w_in"], inp["w_out"])
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    lay.forward_train(x)
    lay.sync()
    with pytest.raises(MoEError):
        lay.stage("x_perm", (t * k, d), torch.bfloat16)
    with pytest.raises(MoEError):
        lay.stage("act", (t * k, f), torch.bfloat16)
    lay.forward(x)
    lay.sync()
    xp = lay.stage("x_perm", (t * k, d), torch.bfloat16)
    perm = lay.stage("perm", (t * k,), torch.int32).long()
    assert torch.equal(xp, x[perm // k])
    lay.close()
