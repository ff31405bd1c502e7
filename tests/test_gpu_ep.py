"""Expert-parallel device path on one GPU: ep_size = 1 loopback through the same NCCL exchange
code (a 1-rank communicator, self send/recv). Multi-rank runs need >1 GPU; their host logic is
covered by tests/test_ep_cpu.py (gloo, 2 and 4 ranks)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs  # noqa: E402


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
