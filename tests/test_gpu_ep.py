"""Expert-parallel device path on one GPU: ep_size = 1 loopback through the same NCCL exchange
code (a 1-rank communicator, self send/recv). Multi-rank runs need >1 GPU; their host logic is
covered by tests/test_ep_cpu.py (gloo, 2 and 4 ranks)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs  # noqa: E402

JOBS = os.cpu_count() or 1


@pytest.mark.parametrize("gemm_ctas", [1, 2])
def test_ep_loopback_matches_oracle(gemm_ctas):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 700, 512, 8, 2, 256
    o = Oracle("port")
    inp = make_inputs(t, d, n, f)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t, gemm_ctas=gemm_ctas),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    lay.ep_init(MoELayer.ep_unique_id())
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    out_ep = lay.ep_forward(x)
    out = lay.forward(x)
    lay.sync()
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"],
                        jobs=os.cpu_count() or 1)
    for res in (out_ep, out):
        dlt = res.float().cpu().numpy().astype(np.float64) - ref
        assert np.linalg.norm(dlt) / np.linalg.norm(ref) <= 1e-2
    lay.close()


def test_ep_loopback_training_matches_oracle():
    """Expert-parallel training step (forward_train + backward_full) through the exchange code with
    a 1-rank communicator: dY pieces out, dX pieces back, dW_r all-reduce."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 600, 256, 8, 2, 256
    o = Oracle("port")
    inp = make_inputs(t, d, n, f)
    g = make_inputs(t, d, 1, f, seed=77, experts=False)["x"]
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    lay.ep_init(MoELayer.ep_unique_id())
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    out = lay.forward_train(x)
    dh, dwr, dwi, dwo = lay.backward_full(torch.from_numpy(g).cuda().to(torch.bfloat16).contiguous(), 0.01, 0.001)
    lay.sync()
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"], jobs=JOBS)

    def rel(a, b):
        return np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b)

    assert rel(out.float().cpu().numpy(), ref) <= 1e-2
    rdh, rdwr, rdwi, rdwo = o.moe_backward_full(inp["x"], inp["w_router"], inp["w_in"], inp["w_out"], g, 0.01, 0.001, k,
                                                jobs=JOBS)
    assert rel(dh.float().cpu().numpy(), rdh) <= 2e-2
    assert rel(dwr.cpu().numpy(), rdwr) <= 2e-2
    assert rel(dwi.cpu().numpy(), rdwi) <= 2e-2
    assert rel(dwo.cpu().numpy(), rdwo) <= 2e-2
    lay.close()


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_ep_stalled_exchange_times_out(transport):
    """A stalled expert-parallel exchange returns CL_ERR_RUN after CL_MOE_EP_TIMEOUT_S (bounded wait
    polling ncclCommGetAsyncError; the communicator is aborted), instead of hanging the caller
    (proj/src/capi.cpp:57-63: failures are status codes). Fresh process: the env is read once."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, CL_MOE_EP_TIMEOUT_S="1", CL_MOE_EP_TEST_STALL_MS="4000")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "helpers", "ep_timeout_check.py"), transport],
                       env=env, capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
