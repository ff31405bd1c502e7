"""GPU parity at the shapes bench.py measures (BASELINE.json configs[1..4] = C2..C5), through the C ABI.

Every case runs the whole layer on the device at the benchmarked shape and checks:
  * routing for ALL tokens bit-exact against the oracle (logits, probs, top-K, weights, counts; the oracle's router is
    cheap on CPU) and the dispatch permutation / expert offsets bit-exact (oracle plan);
  * a sample of output rows against the oracle's per-token compute (orc_expert_ffn per expert, fp64
    accumulation), tolerance as tests/test_gpu_parity.py: rel-F <= 1e-2, max <= 3e-2 max|y| (bf16);
    FP8 vs the qdq-simulated oracle <= 2e-2 rel-F;
  * training (C5 shape): d_hidden and d_combine_w on sampled tokens, and the weight gradients of
    sampled hidden units of three experts (the hot one, a middle one, the coldest non-empty one) —
    the expert FFN restricted to a subset C of its f hidden units is an exact sub-FFN, so
    dW_in[:, C], dW_in[:, f+C] and dW_out[C, :] come from the oracle's expert_ffn_backward on that
    sub-FFN with the same upstream gradient; tolerance rel-F <= 2e-2 (tests/test_gpu_backward.py).
Weights are the device-generated synthetic weights (cl_moe_create_synthetic), read back with
cl_moe_get_weights one expert at a time (the C2 layer is 11 GB in fp32); tokens are the device
synthetic tokens read back. At C2 the GEMM2 L2 tile groups (m_group = 4 < 8 m-tiles per expert)
are active, at C5 the hot expert's GEMM1 groups too.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.oracle import Oracle  # noqa: E402

SEED = 20261018
JOBS = os.cpu_count() or 1


def _layer(T, d, n, k, f, **kw):
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    return MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=T, **kw), seed=SEED)


def _host(t):
    return t.float().cpu().numpy()


def _check_routing(o, lay, x, dec, k, n):
    """All tokens: decision bit-exact; dispatch permutation and offsets bit-exact."""
    wr = lay.router_weights()
    ref = o.route(x, wr, k)
    assert np.array_equal(dec.logits.cpu().numpy(), ref["logits"])
    assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), ref["topk_idx"])
    assert np.array_equal(dec.counts.cpu().numpy(), ref["counts"])
    assert np.array_equal(dec.probs.cpu().numpy(), ref["probs"])
    assert np.array_equal(dec.combine_weights.cpu().numpy(), ref["combine_weights"])
    t = x.shape[0]
    offsets, perm, _ = o.plan(ref["topk_idx"], n)
    assert np.array_equal(lay.stage("offsets", (n + 1,), torch.int32).cpu().numpy(), offsets)
    assert np.array_equal(lay.stage("perm", (t * k,), torch.int32).cpu().numpy(), perm)
    return ref, wr


def _sample(idx, n, per_expert=6, extra=32, seed=0):
    """Tokens covering every expert (first/last of each expert's tokens and a few random) + random."""
    rng = np.random.default_rng(seed)
    pick = set(rng.choice(idx.shape[0], extra, replace=False).tolist())
    for e in range(n):
        toks = np.nonzero((idx == e).any(1))[0]
        if len(toks):
            pick.update([int(toks[0]), int(toks[-1])])
            pick.update(rng.choice(toks, min(per_expert, len(toks)), replace=False).tolist())
    return np.array(sorted(pick))


def _e4m3_round(q):
    """Vectorised E4M3 RNE rounding of fp32 values (the oracle's grid rule): 3
    mantissa bits for |q| >= 2^-6, quantum 2^-9 below, |q| >= 448 clamps. Pinned against
    orc_fp8_qdq in test_e4m3_round_matches_oracle; used so the FP8 reference at d=4096 / f=14336
    is fast."""
    q = np.asarray(q, np.float32)
    a = np.abs(q)
    u = a.view(np.uint32).astype(np.uint64)
    nrm = ((u + 0x7FFFF + ((u >> 20) & 1)) & ~np.uint64(0xFFFFF)).astype(np.uint32).view(np.float32)
    sub = (np.round(a.astype(np.float64) * 512.0) / 512.0).astype(np.float32)
    r = np.where(a >= np.float32(2.0 ** -6), nrm, sub)
    r = np.where(r > 448.0, np.float32(448.0), r)
    return np.copysign(r, q).astype(np.float32)


def _qdq(x, s):
    """orc_fp8_qdq(x, s): q = x / s in fp32, E4M3 rounding, times s in fp32 (s scalar or per column)."""
    return (_e4m3_round((x / s).astype(np.float32)) * s).astype(np.float32)


def test_e4m3_round_matches_oracle():
    o = Oracle("port")
    rng = np.random.default_rng(3)
    q = np.concatenate([rng.standard_normal(200000).astype(np.float32) * np.float32(10.0) ** rng.integers(-4, 3, 200000),
                        np.array([0.0, -0.0, 448.0, 460.0, 464.0, 500.0, 2.0 ** -6, 2.0 ** -7, 2.0 ** -10, 3 * 2.0 ** -10,
                                  -(2.0 ** -9), 1.0625, 1.1875, 240.0, 248.0], np.float32)])
    assert np.array_equal(_e4m3_round(q).view(np.uint32), o.fp8_qdq(q, 1.0).view(np.uint32))
    s = np.float32(0.0123)
    assert np.array_equal(_qdq(q, s).view(np.uint32), o.fp8_qdq(q, float(s)).view(np.uint32))


def _qdq_cols(o, w, s):
    """qdq of every column c of w with scale s[c] (== orc_fp8_qdq per column)."""
    return _qdq(w, s[None, :])


def _win_col_of_packed_row(p, f):
    b, i = p // 256, p % 256
    return np.where(i < 128, b * 128 + i, f + b * 128 + (i - 128))


def _ref_rows(o, lay, x, idx, w, rows, n):
    """Oracle output for tokens `rows`: sum_k w[j,k] * FFN_{idx[j,k]}(x_j), per expert in fp64."""
    d = x.shape[1]
    out = np.zeros((len(rows), d), np.float64)
    pos = {int(j): i for i, j in enumerate(rows)}
    for e in range(n):
        sel = [(pos[int(j)], kk) for j in rows for kk in range(idx.shape[1]) if idx[j, kk] == e]
        if not sel:
            continue
        wi, wo = lay.expert_weights(e)
        xe = x[[rows[i] for i, _ in sel]]
        _, y = o.expert_ffn(xe, wi, wo)
        for (i, kk), yr in zip(sel, y):
            out[i] += np.float64(w[rows[i], kk]) * yr
    return out


def _assert_close(got, ref, rf_tol=1e-2, rm_tol=3e-2):
    dlt = got.astype(np.float64) - ref
    rf = np.linalg.norm(dlt) / np.linalg.norm(ref)
    rm = np.abs(dlt).max() / np.abs(ref).max()
    assert rf <= rf_tol and rm <= rm_tol, (rf, rm)
    return rf, rm


@pytest.mark.parametrize("cfg", [
    pytest.param(dict(T=16384, d=4096, n=16, k=2, f=14336, per=3, extra=16), id="C2"),
    pytest.param(dict(T=8192, d=8192, n=16, k=4, f=12288, per=2, extra=8), id="C3-per-rank"),
])
def test_bf16_layer_at_bench_shape(cfg):
    T, d, n, k, f = cfg["T"], cfg["d"], cfg["n"], cfg["k"], cfg["f"]
    o = Oracle("port")
    lay = _layer(T, d, n, k, f)
    xd = lay.synthetic_tokens(T, SEED)
    out, dec = lay.forward(xd, want_decision=True)
    lay.sync()
    x = _host(xd)
    ref, _ = _check_routing(o, lay, x, dec, k, n)
    rows = _sample(ref["topk_idx"], n, per_expert=cfg["per"], extra=cfg["extra"])
    want = _ref_rows(o, lay, x, ref["topk_idx"], ref["combine_weights"], rows, n)
    rf, rm = _assert_close(_host(out)[rows], want)
    print(f"{len(rows)} sampled rows: rel-F {rf:.2e}, rel-max {rm:.2e}")
    lay.close()


def test_fp8_decode_at_c2_layer_shape():
    """BASELINE configs[3]: expert-aware FP8 at decode batch sizes on the C2 layer (T = 64 takes the
    dense-decode path, T = 512 the sparse one), router through fp8_qdq. One layer,
    one set of quantized reference weights for both batches."""
    from oracle.oracle import router_fp8_sim
    d, n, k, f = 4096, 16, 2, 14336
    o = Oracle("port")
    lay = _layer(2048, d, n, k, f)
    xc = lay.synthetic_tokens(2048, SEED + 1)
    lay.calibrate(xc)
    lay.quantize_fp8()
    _, s_r, _ = lay.router_fp8_scales()
    wr = lay.router_weights()
    s_in, s_mid, wsi_p, wso = lay.fp8_scales()
    wsi = np.empty_like(wsi_p)
    wsi[:, _win_col_of_packed_row(np.arange(2 * f), f)] = wsi_p  # packed row order -> reference columns
    cases = []
    for T in (64, 512):
        xd = lay.synthetic_tokens(T, SEED + T)
        out, dec = lay.forward(xd, want_decision=True)
        lay.sync()
        x = _host(xd)
        rq, _ = router_fp8_sim(o, x, wr, k, s_r)
        assert np.array_equal(dec.logits.cpu().numpy(), rq["logits"]), T
        assert np.array_equal(dec.topk_idx.cpu().numpy().astype(np.int64), rq["topk_idx"]), T
        assert np.array_equal(dec.combine_weights.cpu().numpy(), rq["combine_weights"]), T
        rows = np.arange(T) if T <= 64 else _sample(rq["topk_idx"], n, per_expert=3, extra=16)
        cases.append((T, x, rq, rows, _host(out)[rows]))
    want = {T: np.zeros((len(rows), d), np.float64) for T, _, _, rows, _ in cases}
    for e in range(n):
        wi, wo = lay.expert_weights(e)
        wi_q, wo_q = _qdq_cols(o, wi, wsi[e]).astype(np.float64), _qdq_cols(o, wo, wso[e]).astype(np.float64)
        for T, x, rq, rows, _ in cases:
            sel = [(i, kk) for i, j in enumerate(rows) for kk in range(k) if rq["topk_idx"][j, kk] == e]
            if not sel:
                continue
            xq = _qdq(x[[rows[i] for i, _ in sel]], s_in[e]).astype(np.float64)
            h = xq @ wi_q
            g, u = h[:, :f], h[:, f:]
            aq = _qdq((g / (1.0 + np.exp(-g)) * u).astype(np.float32), s_mid[e]).astype(np.float64)
            y = aq @ wo_q
            for (i, kk), yr in zip(sel, y):
                want[T][i] += np.float64(rq["combine_weights"][rows[i], kk]) * yr
    for T, _, _, rows, got in cases:
        rf, _ = _assert_close(got, want[T], rf_tol=2e-2, rm_tol=1.0)
        print(f"FP8 T={T}: {len(rows)} rows rel-F {rf:.2e}")
    lay.close()


def test_training_at_c5_shape():
    """BASELINE configs[4] on one GPU: T = 65536 skewed tokens (gamma 1.8: expert 0 takes ~1/3 of the
    assignments), forward_train + expert-FFN backward at the C2 layer shape (f = 14336)."""
    T, d, n, k, f = 65536, 4096, 16, 2, 14336
    o = Oracle("port")
    lay = _layer(T, d, n, k, f)
    lay.synthetic_skew(1.8)
    xd = lay.synthetic_tokens(T, SEED, shift=1.0)
    gd = lay.synthetic_tokens(T, SEED + 7)
    out, dec = lay.forward_train(xd, want_decision=True)
    dh, dcw, dwi, dwo = lay.backward(gd)
    lay.sync()
    x, g = _host(xd), _host(gd)
    ref, _ = _check_routing(o, lay, x, dec, k, n)
    counts = ref["counts"]
    assert counts[0] > 0.3 * T * k  # the hot expert
    idx, w = ref["topk_idx"], ref["combine_weights"]
    rows = _sample(idx, n, per_expert=1, extra=8)
    # sampled tokens: output, d_hidden, d_combine_w (full-width expert FFN per sampled row)
    out_ref = np.zeros((len(rows), d), np.float64)
    dh_ref = np.zeros((len(rows), d), np.float64)
    dcw_ref = np.zeros((len(rows), k), np.float64)
    for e in range(n):
        sel = [(i, kk) for i, j in enumerate(rows) for kk in range(k) if idx[j, kk] == e]
        if not sel:
            continue
        wi, wo = lay.expert_weights(e)
        xe = x[[rows[i] for i, _ in sel]]
        dy = np.stack([w[rows[i], kk] * g[rows[i]] for i, kk in sel]).astype(np.float32)
        dx, _, _ = o.expert_ffn_backward(xe, wi, wo, dy)
        _, y = o.expert_ffn(xe, wi, wo)
        for (i, kk), dxr, yr in zip(sel, dx, y):
            out_ref[i] += np.float64(w[rows[i], kk]) * yr
            dh_ref[i] += dxr
            dcw_ref[i, kk] = np.dot(g[rows[i]].astype(np.float64), yr.astype(np.float64))
    _assert_close(_host(out)[rows], out_ref)
    _assert_close(_host(dh)[rows], dh_ref, rf_tol=2e-2, rm_tol=5e-2)
    _assert_close(dcw.cpu().numpy()[rows], dcw_ref, rf_tol=2e-2, rm_tol=5e-2)
    # weight gradients of sampled hidden units: exact sub-FFN on the hidden units C
    order = np.argsort(counts)
    cold = int(order[np.nonzero(counts[order] > 0)[0][0]])
    rng = np.random.default_rng(1)
    C = np.sort(rng.choice(f, 16, replace=False))
    for e in sorted({0, int(order[n // 2]), cold}):
        tok, slot = np.nonzero(idx == e)
        wi, wo = lay.expert_weights(e)
        wi_sub = np.ascontiguousarray(np.concatenate([wi[:, C], wi[:, f + C]], axis=1))
        wo_sub = np.ascontiguousarray(wo[C])
        dy = (w[tok, slot][:, None] * g[tok]).astype(np.float32)
        _, dwi_ref, dwo_ref = o.expert_ffn_backward(x[tok], wi_sub, wo_sub, dy)
        got_wi = np.concatenate([dwi[e][:, C].cpu().numpy(), dwi[e][:, f + C].cpu().numpy()], axis=1)
        got_wo = dwo[e][C].cpu().numpy()
        _assert_close(got_wi, dwi_ref.astype(np.float64), rf_tol=2e-2, rm_tol=5e-2)
        _assert_close(got_wo, dwo_ref.astype(np.float64), rf_tol=2e-2, rm_tol=5e-2)
    lay.close()
