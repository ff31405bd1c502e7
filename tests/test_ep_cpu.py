"""Expert-parallel host logic on CPU: the receive layout (C ABI, no GPU) and a 2-rank gloo run
of the full EP data movement (route -> plan -> piece exchange -> expert FFN -> reverse exchange
-> combine) with the oracle as the per-rank expert compute, checked bit-for-bit against the
single-process oracle layer."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2509_09121_b200.moe import ep_layout  # noqa: E402


def test_layout_partitions_receive_buffer():
    rng = np.random.default_rng(0)
    for r in (1, 2, 4, 8):
        n = 16
        counts = rng.integers(0, 50, (r, n))
        for rank in range(r):
            loc, piece, tot = ep_layout(counts, rank)
            nl = n // r
            mine = counts[:, rank * nl:(rank + 1) * nl]  # [src, local expert]
            assert tot == mine.sum()
            assert loc[0] == 0 and loc[-1] == tot
            assert np.array_equal(np.diff(loc), mine.sum(0))
            # pieces in (expert, source) order tile [0, tot) exactly
            starts = piece.ravel()
            sizes = mine.T.ravel()
            assert np.array_equal(starts, np.concatenate([[0], np.cumsum(sizes)[:-1]]))


def test_layout_rejects_bad_arguments():
    from paper_2509_09121_b200.moe import MoEConfigError
    with pytest.raises(MoEConfigError):
        ep_layout(np.zeros((3, 16), np.int64), 0)  # 16 experts not divisible by 3 ranks
    with pytest.raises(MoEConfigError):
        ep_layout(np.zeros((2, 16), np.int64), 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ep_worker(rank, world, port, t, d, n, k, f, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle, make_inputs
    o = Oracle("port")
    full = make_inputs(t * world, d, n, f)
    nl = n // world
    xs = full["x"][rank * t:(rank + 1) * t]
    r = o.route(xs, full["w_router"], k)
    idx, w = r["topk_idx"], r["combine_weights"]
    offsets, perm, inv = o.plan(idx, n)
    xperm = xs[perm // k]
    counts = np.diff(offsets).astype(np.int64)
    allc = [torch.zeros(n, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, torch.from_numpy(counts))
    cmat = torch.stack(allc).numpy()
    loc, piece, tot = ep_layout(cmat, rank)
    recv = np.zeros((tot, d), np.float32)
    reqs = []
    # dispatch exchange (gloo p2p)
    for dst in range(world):
        for e in range(nl):
            g = dst * nl + e
            cnt = cmat[rank, g]
            if cnt:
                buf = torch.from_numpy(np.ascontiguousarray(xperm[offsets[g]:offsets[g] + cnt]))
                if dst == rank:
                    recv[piece[e, rank]:piece[e, rank] + cnt] = buf.numpy()
                else:
                    reqs.append(dist.isend(buf, dst, tag=g))
    bufs = []
    for e in range(nl):
        for src in range(world):
            cnt = cmat[src, rank * nl + e]
            if cnt and src != rank:
                b = torch.zeros(cnt, d)
                reqs.append(dist.irecv(b, src, tag=rank * nl + e))
                bufs.append((e, src, b))
    for q in reqs:
        q.wait()
    for e, src, b in bufs:
        recv[piece[e, src]:piece[e, src] + len(b)] = b.numpy()
    # local experts
    yrecv = np.zeros_like(recv)
    for e in range(nl):
        g = rank * nl + e
        a, b = loc[e], loc[e + 1]
        if b > a:
            _, yrecv[a:b] = o.expert_ffn(recv[a:b], full["w_in"][g], full["w_out"][g])
    # reverse exchange
    y = np.zeros((t * k, d), np.float32)
    reqs, bufs = [], []
    for e in range(nl):
        for src in range(world):
            cnt = cmat[src, rank * nl + e]
            if cnt:
                chunk = np.ascontiguousarray(yrecv[piece[e, src]:piece[e, src] + cnt])
                if src == rank:
                    g = rank * nl + e
                    y[offsets[g]:offsets[g] + cnt] = chunk
                else:
                    reqs.append(dist.isend(torch.from_numpy(chunk), src, tag=1000 + rank * nl + e))
    for srcr in range(world):
        for e in range(nl):
            g = srcr * nl + e
            cnt = cmat[rank, g]
            if cnt and srcr != rank:
                b = torch.zeros(cnt, d)
                reqs.append(dist.irecv(b, srcr, tag=1000 + g))
                bufs.append((g, b))
    for q in reqs:
        q.wait()
    for g, b in bufs:
        y[offsets[g]:offsets[g] + len(b)] = b.numpy()
    # combine at the source, expert order like the reference's add chain
    out = np.zeros((t, d), np.float32)
    order = np.argsort(idx, axis=1, kind="stable")
    for j in range(t):
        for kk in order[j]:
            out[j] = out[j] + (y[inv[j * k + kk]] * w[j, kk]).astype(np.float32)
    np.save(os.path.join(result_dir, f"out{rank}.npy"), out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k", [(2, 8, 2), (4, 8, 2)])
def test_ep_gloo_matches_single_process_oracle(tmp_path, world, n, k):
    t, d, f = 48, 64, 32
    mp.spawn(_ep_worker, args=(world, _free_port(), t, d, n, k, f, str(tmp_path)), nprocs=world, join=True)
    from oracle.oracle import Oracle, make_inputs
    o = Oracle("port")
    full = make_inputs(t * world, d, n, f)
    r = o.route(full["x"], full["w_router"], k)
    ref = o.moe_forward(full["x"], full["w_in"], full["w_out"], r["topk_idx"], r["combine_weights"])
    got = np.concatenate([np.load(tmp_path / f"out{i}.npy") for i in range(world)])
    assert np.array_equal(got, ref)


def _exchange(rank, world, nl, cmat, offsets, piece, src, dst_rows, d, to_experts, tag0):
    """gloo p2p restatement of cl_moe's ep_exchange (csrc/capi.cu)."""
    dst = np.zeros((dst_rows, d), np.float32)
    reqs, bufs = [], []
    if to_experts:
        for r in range(world):
            for e in range(nl):
                g = r * nl + e
                cnt = cmat[rank, g]
                if not cnt:
                    continue
                chunk = np.ascontiguousarray(src[offsets[g]:offsets[g] + cnt])
                if r == rank:
                    dst[piece[e, rank]:piece[e, rank] + cnt] = chunk
                else:
                    reqs.append(dist.isend(torch.from_numpy(chunk), r, tag=tag0 + g))
        for e in range(nl):
            for s in range(world):
                cnt = cmat[s, rank * nl + e]
                if cnt and s != rank:
                    b = torch.zeros(cnt, d)
                    reqs.append(dist.irecv(b, s, tag=tag0 + rank * nl + e))
                    bufs.append((piece[e, s], b))
    else:
        for e in range(nl):
            for s in range(world):
                cnt = cmat[s, rank * nl + e]
                if not cnt:
                    continue
                chunk = np.ascontiguousarray(src[piece[e, s]:piece[e, s] + cnt])
                g = rank * nl + e
                if s == rank:
                    dst[offsets[g]:offsets[g] + cnt] = chunk
                else:
                    reqs.append(dist.isend(torch.from_numpy(chunk), s, tag=tag0 + g))
        for r in range(world):
            for e in range(nl):
                g = r * nl + e
                cnt = cmat[rank, g]
                if cnt and r != rank:
                    b = torch.zeros(cnt, d)
                    reqs.append(dist.irecv(b, r, tag=tag0 + g))
                    bufs.append((offsets[g], b))
    for q in reqs:
        q.wait()
    for start, b in bufs:
        dst[start:start + len(b)] = b.numpy()
    return dst


def _ep_bwd_worker(rank, world, port, t, d, n, k, f, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle, make_inputs
    o = Oracle("port")
    full = make_inputs(t * world, d, n, f)
    gfull = make_inputs(t * world, d, 1, f, seed=31, experts=False)["x"]
    nl = n // world
    xs = full["x"][rank * t:(rank + 1) * t]
    gs = gfull[rank * t:(rank + 1) * t]
    r = o.route(xs, full["w_router"], k)
    idx, w = r["topk_idx"], r["combine_weights"]
    offsets, perm, inv = o.plan(idx, n)
    allc = [torch.zeros(n, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, torch.from_numpy(np.diff(offsets).astype(np.int64)))
    cmat = torch.stack(allc).numpy()
    loc, piece, tot = ep_layout(cmat, rank)
    # forward: y (unweighted) back at the source
    x_recv = _exchange(rank, world, nl, cmat, offsets, piece, xs[perm // k], tot, d, True, 0)
    y_recv = np.zeros_like(x_recv)
    for e in range(nl):
        a, b = loc[e], loc[e + 1]
        if b > a:
            _, y_recv[a:b] = o.expert_ffn(x_recv[a:b], full["w_in"][rank * nl + e], full["w_out"][rank * nl + e])
    y = _exchange(rank, world, nl, cmat, offsets, piece, y_recv, t * k, d, False, 10000)
    # backward at the source: dY = w * dOut[token], d_cw = <dOut, Y> (fp64 sum like mul_rowwise bwd)
    wslot = w.ravel()[perm]
    dy_src = (gs[perm // k] * wslot[:, None]).astype(np.float32)
    dcw = np.zeros(t * k, np.float32)
    dcw[perm] = (gs[perm // k].astype(np.float64) * y.astype(np.float64)).sum(1).astype(np.float32)
    dy_recv = _exchange(rank, world, nl, cmat, offsets, piece, dy_src, tot, d, True, 20000)
    dx_recv = np.zeros_like(x_recv)
    dwi = np.zeros((nl, d, 2 * f), np.float32)
    dwo = np.zeros((nl, f, d), np.float32)
    for e in range(nl):
        a, b = loc[e], loc[e + 1]
        if b > a:
            dx_recv[a:b], dwi[e], dwo[e] = o.expert_ffn_backward(x_recv[a:b], full["w_in"][rank * nl + e],
                                                                 full["w_out"][rank * nl + e], dy_recv[a:b])
    dx = _exchange(rank, world, nl, cmat, offsets, piece, dx_recv, t * k, d, False, 30000)
    dh = np.zeros((t, d), np.float32)
    for j in range(t):
        for kk in range(k):
            dh[j] = dh[j] + dx[inv[j * k + kk]]
    np.savez(os.path.join(result_dir, f"bwd{rank}.npz"), dh=dh, dcw=dcw.reshape(t, k), dwi=dwi, dwo=dwo)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k", [(2, 8, 2), (4, 8, 2)])
def test_ep_gloo_backward_matches_single_process_oracle(tmp_path, world, n, k):
    t, d, f = 40, 64, 32
    mp.spawn(_ep_bwd_worker, args=(world, _free_port(), t, d, n, k, f, str(tmp_path)), nprocs=world, join=True)
    from oracle.oracle import Oracle, make_inputs
    o = Oracle("port")
    full = make_inputs(t * world, d, n, f)
    g = make_inputs(t * world, d, 1, f, seed=31, experts=False)["x"]
    r = o.route(full["x"], full["w_router"], k)
    rdh, rdcw, rdwi, rdwo = o.moe_backward(full["x"], full["w_in"], full["w_out"], r["topk_idx"], r["combine_weights"], g)
    parts = [np.load(tmp_path / f"bwd{i}.npz") for i in range(world)]
    assert np.array_equal(np.concatenate([p_["dh"] for p_ in parts]), rdh)
    assert np.array_equal(np.concatenate([p_["dcw"] for p_ in parts]), rdcw)
    nl = n // world
    for i, p_ in enumerate(parts):
        for e in range(nl):
            cnt = int((r["topk_idx"] == i * nl + e).sum())
            if cnt:
                assert np.array_equal(p_["dwi"][e], rdwi[i * nl + e]), (i, e)
                assert np.array_equal(p_["dwo"][e], rdwo[i * nl + e]), (i, e)
