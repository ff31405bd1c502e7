"""Peer-memory (NVLink) expert-parallel transport on one GPU.

* R-rank groups emulated in one process (cl_moe_ep_group_forward): the production layout,
  dispatch (stores into the owners' receive buffers) and GEMM2 epilogue (stores into the sources'
  return buffers) kernels, with the other handles' buffers as peer addresses, phase by phase so no
  kernel waits on another. Output must be bit-identical to the single-GPU layer on each rank's
  batch (a row's GEMM result does not depend on which rows share its tile).
* ep_size = 1 through cl_moe_ep_peer_init with a real 1-rank communicator (NCCL counts
  all-gather and barriers, self "peer" = local buffers)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.oracle import Oracle, make_inputs  # noqa: E402

JOBS = os.cpu_count() or 1


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16).contiguous()


# (the last two: per-rank batches large enough for the fp64 tensor-core router and its finish tiles)
@pytest.mark.parametrize("R,n,k,ts,gemm_ctas", [(2, 8, 2, (300, 517), 1), (2, 8, 2, (1024, 900), 2),
                                                 (4, 16, 4, (300, 1, 517, 64), 1), (4, 16, 2, (640, 640, 3, 700), 2),
                                                 (8, 16, 2, (128,) * 8, 1), (2, 8, 2, (4096, 3000), 2),
                                                 (4, 16, 2, (5000, 3100, 2500, 4000), 2)])
def test_group_forward_bit_identical_to_single_gpu(R, n, k, ts, gemm_ctas):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer, ep_group_forward
    d, f = 512, 256
    T = sum(ts)
    inp = make_inputs(T, d, n, f)
    nl = n // R
    cap = max(ts)
    full = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=cap, gemm_ctas=gemm_ctas),
                    inp["w_router"], inp["w_in"], inp["w_out"])
    ranks = [MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=cap, gemm_ctas=gemm_ctas,
                                ep_size=R, ep_rank=r),
                      inp["w_router"], inp["w_in"][r * nl:(r + 1) * nl], inp["w_out"][r * nl:(r + 1) * nl])
             for r in range(R)]
    xs, a = [], 0
    for t in ts:
        xs.append(_dev(inp["x"][a:a + t]))
        a += t
    outs = ep_group_forward(ranks, xs)
    for r in range(R):
        ranks[r].sync()
        assert torch.equal(outs[r], full.forward(xs[r])), f"rank {r}"
    # twice: buffers are reused across forwards
    outs2 = ep_group_forward(ranks, xs)
    assert all(torch.equal(a_, b_) for a_, b_ in zip(outs, outs2))
    if R == 2:
        o = Oracle("port")
        rr = o.route(inp["x"][:ts[0]], inp["w_router"], k)
        ref = o.moe_forward(inp["x"][:ts[0]], inp["w_in"], inp["w_out"], rr["topk_idx"], rr["combine_weights"],
                            jobs=JOBS)
        dl = outs[0].float().cpu().numpy().astype(np.float64) - ref
        assert np.linalg.norm(dl) / np.linalg.norm(ref) <= 1e-2


def test_group_forward_skewed_routing():
    """One expert (owned by rank 0) receives most rows from every rank."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer, ep_group_forward
    R, n, k, d, f, t = 4, 16, 2, 256, 256, 400
    inp = make_inputs(R * t, d, n, f, skew=2.0)
    nl = n // R
    full = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                    inp["w_router"], inp["w_in"], inp["w_out"])
    ranks = [MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t, ep_size=R, ep_rank=r),
                      inp["w_router"], inp["w_in"][r * nl:(r + 1) * nl], inp["w_out"][r * nl:(r + 1) * nl])
             for r in range(R)]
    xs = [_dev(inp["x"][r * t:(r + 1) * t]) for r in range(R)]
    outs = ep_group_forward(ranks, xs)
    for r in range(R):
        assert torch.equal(outs[r], full.forward(xs[r]))


def test_group_forward_rejects_mismatched_group():
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer, MoEConfigError, ep_group_forward
    d, n, f = 256, 8, 256
    inp = make_inputs(8, d, n, f)
    a = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=2, d_ff=f, max_tokens=8, ep_size=2, ep_rank=0),
                 inp["w_router"], inp["w_in"][:4], inp["w_out"][:4])
    b = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=2, d_ff=f, max_tokens=8, ep_size=2, ep_rank=0),
                 inp["w_router"], inp["w_in"][:4], inp["w_out"][:4])
    with pytest.raises(MoEConfigError):
        ep_group_forward([a, b], [_dev(inp["x"]), _dev(inp["x"])])


def test_peer_transport_single_rank_nccl():
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 700, 512, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    ref = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    lay.ep_init(MoELayer.ep_unique_id())
    lay.ep_peer_init()
    x = _dev(inp["x"])
    for _ in range(2):
        out = lay.ep_forward(x)
        lay.sync()
        assert torch.equal(out, ref.forward(x))
    counts = Oracle("port").route(inp["x"], inp["w_router"], k)["counts"]
    assert np.array_equal(lay.ep_last_counts(), counts[None, :])


@pytest.mark.parametrize("R,n,k,ts", [(2, 8, 2, (300, 517)), (4, 16, 4, (256, 1, 700, 64))])
def test_group_forward_fp8_bit_identical_to_single_gpu(R, n, k, ts):
    """Expert-parallel FP8: the source quantizes each dispatched row with its owner's GEMM1-input
    scale (global table), owners run the e4m3 GEMMs; bit-identical to the single-GPU FP8 layer."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer, ep_group_forward
    d, f = 512, 256
    inp = make_inputs(sum(ts), d, n, f)
    nl = n // R
    cap = max(ts)
    full = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=sum(ts)),
                    inp["w_router"], inp["w_in"], inp["w_out"])
    xall = _dev(inp["x"])
    full.calibrate(xall)
    full.quantize_fp8()
    s_in, s_mid, _, _ = full.fp8_scales()
    s_r = full.router_fp8_scales()[1]  # every rank routes with the same router activation scale
    ranks = []
    for r in range(R):
        lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=cap, ep_size=R, ep_rank=r),
                       inp["w_router"], inp["w_in"][r * nl:(r + 1) * nl], inp["w_out"][r * nl:(r + 1) * nl])
        lay.quantize_fp8(s_in, s_mid[r * nl:(r + 1) * nl], router_act_scale=s_r)
        ranks.append(lay)
    xs, a = [], 0
    for t in ts:
        xs.append(_dev(inp["x"][a:a + t]))
        a += t
    outs = ep_group_forward(ranks, xs)
    for r in range(R):
        assert torch.equal(outs[r], full.forward(xs[r])), f"rank {r}"


@pytest.mark.parametrize("peer", [False, True])
def test_ep_fp8_calibration_single_rank_nccl(peer):
    """EP calibration (source-side per-expert maxima, all-reduced by quantize) gives the same scales
    as the single-GPU calibration; the FP8 EP forward then matches the single-GPU FP8 layer
    (bit-identical over the peer transport, within bf16 rounding of the combine over NCCL)."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 600, 512, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    x = _dev(inp["x"])
    ref = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    ref.calibrate(x)
    ref.quantize_fp8()
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    lay.ep_init(MoELayer.ep_unique_id())
    if peer:
        lay.ep_peer_init()
    lay.calibrate(x)
    lay.quantize_fp8()
    for a_, b_ in zip(lay.fp8_scales(), ref.fp8_scales()):
        assert np.array_equal(a_, b_)
    out, want = lay.ep_forward(x), ref.forward(x)
    lay.sync()
    if peer:
        assert torch.equal(out, want)
    else:
        dl = (out.float() - want.float()).abs().max().item()
        assert dl <= 2e-2 * want.float().abs().max().item()


@pytest.mark.parametrize("R,n,k,t", [(2, 8, 2, 300), (4, 16, 2, 200), (2, 8, 2, 3000)])
def test_group_train_step_bit_identical_to_single_gpu(R, n, k, t):
    """EP training over the peer transport (emulated group): forward_train + expert-FFN backward.
    Ranks hold consecutive token slices, so each expert's receive layout is the single-GPU row
    order of the concatenated batch: outputs, d_hidden, d_combine_w AND the weight gradients are
    bit-identical to the single-GPU layer on the whole batch."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer, ep_group_train_step
    d, f = 256, 256
    inp = make_inputs(R * t, d, n, f)
    g = make_inputs(R * t, d, 1, f, seed=99, experts=False)["x"]
    nl = n // R
    full = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=R * t, gemm_ctas=2),
                    inp["w_router"], inp["w_in"], inp["w_out"])
    out_f = full.forward_train(_dev(inp["x"]))
    dh_f, dcw_f, dwi_f, dwo_f = full.backward(_dev(g))
    full.sync()
    ranks = [MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t, gemm_ctas=2, ep_size=R,
                                ep_rank=r),
                      inp["w_router"], inp["w_in"][r * nl:(r + 1) * nl], inp["w_out"][r * nl:(r + 1) * nl])
             for r in range(R)]
    res = ep_group_train_step(ranks, [_dev(inp["x"][r * t:(r + 1) * t]) for r in range(R)],
                              [_dev(g[r * t:(r + 1) * t]) for r in range(R)])
    for r in range(R):
        out, dh, dcw, dwi, dwo = res[r]
        sl = slice(r * t, (r + 1) * t)
        assert torch.equal(out, out_f[sl]), f"out rank {r}"
        assert torch.equal(dh, dh_f[sl]), f"d_hidden rank {r}"
        assert torch.equal(dcw, dcw_f[sl]), f"d_combine_w rank {r}"
        assert torch.equal(dwi, dwi_f[r * nl:(r + 1) * nl]), f"dW_in rank {r}"
        assert torch.equal(dwo, dwo_f[r * nl:(r + 1) * nl]), f"dW_out rank {r}"


def test_peer_transport_training_single_rank_nccl():
    """ep_size = 1 with a real communicator over the peer transport: training matches the
    single-GPU layer bit for bit (full backward incl. the router, dW_r all-reduced)."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 400, 256, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    g = make_inputs(t, d, 1, f, seed=5, experts=False)["x"]
    ref = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    lay.ep_init(MoELayer.ep_unique_id())
    lay.ep_peer_init()
    x, gd = _dev(inp["x"]), _dev(g)
    for _ in range(2):
        a = lay.forward_train(x)
        ga = lay.backward_full(gd, 0.01, 0.001)
        b = ref.forward_train(x)
        gb = ref.backward_full(gd, 0.01, 0.001)
        lay.sync()
        assert torch.equal(a, b)
        for u, v in zip(ga, gb):
            assert torch.equal(u, v)


@pytest.fixture
def _overlap():
    """CL_MOE_EP_OVERLAP=1 (read per call): dispatch overlapped with the owners' GEMM1 — no barrier
    between them; GEMM1's producer waits on per-expert arrival counters the sources' dispatch
    kernels bump with system-scope releases."""
    os.environ["CL_MOE_EP_OVERLAP"] = "1"
    yield
    del os.environ["CL_MOE_EP_OVERLAP"]


@pytest.mark.parametrize("R,n,k,ts,gemm_ctas", [(2, 8, 2, (300, 517), 1), (4, 16, 4, (300, 1, 517, 64), 2),
                                                 (8, 16, 2, (6000,) * 8, 2)])
def test_group_forward_dispatch_overlap_bit_identical(_overlap, R, n, k, ts, gemm_ctas):
    """The counters' bookkeeping (targets from the all-gathered counts x the sources' column
    slices, epochs across forwards) on the emulated group: every GEMM1 finds its rows complete and
    the outputs stay bit-identical to the single-GPU layer, over three forwards (running counters).
    In the emulation every rank's dispatch precedes every GEMM1, so the waits never block here —
    the waiting itself only happens across real GPUs."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer, ep_group_forward
    d, f = 512, 256
    inp = make_inputs(sum(ts), d, n, f)
    nl = n // R
    cap = max(ts)
    full = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=cap, gemm_ctas=gemm_ctas),
                    inp["w_router"], inp["w_in"], inp["w_out"])
    ranks = [MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=cap, gemm_ctas=gemm_ctas,
                                ep_size=R, ep_rank=r),
                      inp["w_router"], inp["w_in"][r * nl:(r + 1) * nl], inp["w_out"][r * nl:(r + 1) * nl])
             for r in range(R)]
    xs, a = [], 0
    for t in ts:
        xs.append(_dev(inp["x"][a:a + t]))
        a += t
    for _ in range(3):
        outs = ep_group_forward(ranks, xs)
        for r in range(R):
            ranks[r].sync()  # also: no "rows did not arrive" error
            assert torch.equal(outs[r], full.forward(xs[r])), f"rank {r}"


def test_peer_transport_dispatch_overlap_single_rank_nccl(_overlap):
    """The real NCCL + CUDA-IPC path (counters mapped through the IPC handle exchange) at ep_size 1,
    forward and a training step."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    t, d, n, k, f = 700, 512, 8, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    ref = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t),
                   inp["w_router"], inp["w_in"], inp["w_out"])
    lay.ep_init(MoELayer.ep_unique_id())
    lay.ep_peer_init()
    x = _dev(inp["x"])
    for _ in range(3):
        out = lay.ep_forward(x)
        lay.sync()
        assert torch.equal(out, ref.forward(x))
    g = _dev(make_inputs(t, d, 1, f, seed=77, experts=False)["x"])
    lay.forward_train(x)
    ref.forward_train(x)
    a_ = lay.backward(g)
    b_ = ref.backward(g)
    lay.sync()
    for u, v in zip(a_, b_):
        assert torch.equal(u, v)
