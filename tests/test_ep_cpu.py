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


# ---- peer-memory (NVLink) transport: layout consistency and a gloo restatement of the one-sided
# stores (cl_moe_ep_peer_layout / ep_peer_layout_kernel, csrc/ep.cuh) ----

def test_peer_layout_agrees_across_ranks():
    """Every source's independently computed dispatch row equals the owner's receive-piece start;
    every owner's return row equals the piece start in the source's permutation."""
    from paper_2509_09121_b200.moe import ep_peer_layout
    rng = np.random.default_rng(3)
    for world, n in ((1, 8), (2, 8), (4, 16), (8, 16), (8, 64)):
        nl = n // world
        counts = rng.integers(0, 40, (world, n))
        counts[rng.random((world, n)) < 0.2] = 0  # empty pieces
        recv = [ep_layout(counts, o) for o in range(world)]
        peer = [ep_peer_layout(counts, r) for r in range(world)]
        for s in range(world):
            disp, _, _ = peer[s]
            src_off = np.concatenate([[0], np.cumsum(counts[s])])
            for g in range(n):
                o, e = divmod(g, nl)
                assert disp[g] == recv[o][1][e, s]
        for o in range(world):
            _, ret, loc = peer[o]
            assert np.array_equal(loc, recv[o][0])
            for e in range(nl):
                for s in range(world):
                    assert ret[e, s] == np.cumsum(np.concatenate([[0], counts[s]]))[o * nl + e]


def _ep_peer_worker(rank, world, port, t, d, n, k, f, result_dir):
    """One-sided stores restated over gloo: each writer computes the destination rows itself
    (from ep_peer_layout) and ships (rows, data); the target only scatters. A layout mismatch
    would overwrite or leave holes, caught by the hole check and the bit-exact comparison."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle, make_inputs
    from paper_2509_09121_b200.moe import ep_peer_layout
    o = Oracle("port")
    full = make_inputs(t * world, d, n, f)
    nl = n // world
    xs = full["x"][rank * t:(rank + 1) * t]
    r = o.route(xs, full["w_router"], k)
    idx, w = r["topk_idx"], r["combine_weights"]
    offsets, perm, inv = o.plan(idx, n)
    counts = np.diff(offsets).astype(np.int64)
    allc = [torch.zeros(n, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, torch.from_numpy(counts))
    cmat = torch.stack(allc).numpy()
    disp, ret, loc = ep_peer_layout(cmat, rank)

    def one_sided(stores, rows):
        """stores[dst] = (row indices, data); returns this rank's buffer after everyone's stores."""
        sent = [None] * world
        dist.all_gather_object(sent, stores)
        buf = np.full((rows, d), np.nan, np.float32)
        for s in range(world):
            ridx, data = sent[s][rank]
            assert np.isnan(buf[ridx]).all(), "two writers hit the same row"
            buf[ridx] = data
        return buf

    # dispatch: row r of expert g (rank-in-expert r - offsets[g]) -> owner row disp[g] + that rank
    stores = [([], []) for _ in range(world)]
    for g in range(n):
        for j in range(offsets[g], offsets[g + 1]):
            stores[g // nl][0].append(disp[g] + j - offsets[g])
            stores[g // nl][1].append(xs[perm[j] // k])
    stores = [(np.array(a, np.int64), np.array(b, np.float32).reshape(-1, d)) for a, b in stores]
    recv = one_sided(stores, loc[-1])
    assert not np.isnan(recv).any(), "receive buffer has holes"
    # experts, then the GEMM2-epilogue stores: received row loc-piece (e, s) + j -> s's row ret[e, s] + j
    yrecv = np.zeros_like(recv)
    for e in range(nl):
        a, b = loc[e], loc[e + 1]
        if b > a:
            _, yrecv[a:b] = o.expert_ffn(recv[a:b], full["w_in"][rank * nl + e], full["w_out"][rank * nl + e])
    stores = [([], []) for _ in range(world)]
    row = 0
    for e in range(nl):
        for s in range(world):
            cnt = cmat[s, rank * nl + e]
            stores[s][0].extend(range(ret[e, s], ret[e, s] + cnt))
            stores[s][1].extend(yrecv[row:row + cnt])
            row += cnt
    stores = [(np.array(a, np.int64), np.array(b, np.float32).reshape(-1, d)) for a, b in stores]
    y = one_sided(stores, t * k)
    assert not np.isnan(y).any(), "return buffer has holes"
    out = np.zeros((t, d), np.float32)
    order = np.argsort(idx, axis=1, kind="stable")
    for j in range(t):
        for kk in order[j]:
            out[j] = out[j] + (y[inv[j * k + kk]] * w[j, kk]).astype(np.float32)
    np.save(os.path.join(result_dir, f"out{rank}.npy"), out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k", [(2, 8, 2), (4, 16, 4)])
def test_ep_peer_transport_gloo_matches_single_process_oracle(tmp_path, world, n, k):
    t, d, f = 40, 64, 32
    mp.spawn(_ep_peer_worker, args=(world, _free_port(), t, d, n, k, f, str(tmp_path)), nprocs=world, join=True)
    from oracle.oracle import Oracle, make_inputs
    o = Oracle("port")
    full = make_inputs(t * world, d, n, f)
    r = o.route(full["x"], full["w_router"], k)
    ref = o.moe_forward(full["x"], full["w_in"], full["w_out"], r["topk_idx"], r["combine_weights"])
    got = np.concatenate([np.load(tmp_path / f"out{i}.npy") for i in range(world)])
    assert np.array_equal(got, ref)


def _one_sided(rank, world, stores, rows, d):
    """stores[dst] = (row indices, data): every writer ships rows it addressed itself; the target
    only scatters (and checks that no row is written twice or left empty)."""
    sent = [None] * world
    dist.all_gather_object(sent, stores)
    buf = np.full((rows, d), np.nan, np.float32)
    for s in range(world):
        ridx, data = sent[s][rank]
        assert np.isnan(buf[ridx]).all(), "two writers hit the same row"
        buf[ridx] = data
    assert not np.isnan(buf).any(), "buffer has holes"
    return buf


def _pack(stores):
    return [(np.array(a, np.int64), np.array(b, np.float32).reshape(-1, stores[0][2])) for a, b, _ in stores]


def _ep_peer_bwd_worker(rank, world, port, t, d, n, k, f, result_dir):
    """Training over the peer transport, restated with one-sided stores: dispatch (x rows) and
    the combine-backward kernel (dY rows) write at disp[g] + rank-in-expert of the owner; the
    GEMM2 epilogue (Y rows) and the dgrad-2 epilogue (dX rows) write at ret[e, s] + j of the
    source -- every address computed by the writer from cl_moe_ep_peer_layout."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle, make_inputs
    from paper_2509_09121_b200.moe import ep_peer_layout
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
    disp, ret, loc = ep_peer_layout(cmat, rank)

    def to_owners(rows_src):  # source-permutation rows -> owners' receive buffers
        st = [([], [], d) for _ in range(world)]
        for g in range(n):
            for j in range(offsets[g], offsets[g + 1]):
                st[g // nl][0].append(disp[g] + j - offsets[g])
                st[g // nl][1].append(rows_src[j])
        return _one_sided(rank, world, _pack(st), loc[-1], d)

    def to_sources(rows_recv):  # receive-layout rows -> sources' permutations
        st = [([], [], d) for _ in range(world)]
        row = 0
        for e in range(nl):
            for s in range(world):
                cnt = cmat[s, rank * nl + e]
                st[s][0].extend(range(ret[e, s], ret[e, s] + cnt))
                st[s][1].extend(rows_recv[row:row + cnt])
                row += cnt
        return _one_sided(rank, world, _pack(st), t * k, d)

    x_recv = to_owners(xs[perm // k])
    y_recv = np.zeros_like(x_recv)
    for e in range(nl):
        a, b = loc[e], loc[e + 1]
        if b > a:
            _, y_recv[a:b] = o.expert_ffn(x_recv[a:b], full["w_in"][rank * nl + e], full["w_out"][rank * nl + e])
    y = to_sources(y_recv)  # unweighted Y at the source (training keeps it for d(combine w))
    wslot = w.ravel()[perm]
    dy_src = (gs[perm // k] * wslot[:, None]).astype(np.float32)
    dcw = np.zeros(t * k, np.float32)
    dcw[perm] = (gs[perm // k].astype(np.float64) * y.astype(np.float64)).sum(1).astype(np.float32)
    dy_recv = to_owners(dy_src)
    dx_recv = np.zeros_like(x_recv)
    dwi = np.zeros((nl, d, 2 * f), np.float32)
    dwo = np.zeros((nl, f, d), np.float32)
    for e in range(nl):
        a, b = loc[e], loc[e + 1]
        if b > a:
            dx_recv[a:b], dwi[e], dwo[e] = o.expert_ffn_backward(x_recv[a:b], full["w_in"][rank * nl + e],
                                                                 full["w_out"][rank * nl + e], dy_recv[a:b])
    dx = to_sources(dx_recv)
    dh = np.zeros((t, d), np.float32)
    for j in range(t):
        for kk in range(k):
            dh[j] = dh[j] + dx[inv[j * k + kk]]
    np.savez(os.path.join(result_dir, f"pbwd{rank}.npz"), dh=dh, dcw=dcw.reshape(t, k), dwi=dwi, dwo=dwo)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k", [(2, 8, 2), (4, 16, 2)])
def test_ep_peer_transport_backward_gloo_matches_single_process_oracle(tmp_path, world, n, k):
    t, d, f = 32, 64, 32
    mp.spawn(_ep_peer_bwd_worker, args=(world, _free_port(), t, d, n, k, f, str(tmp_path)), nprocs=world, join=True)
    from oracle.oracle import Oracle, make_inputs
    o = Oracle("port")
    full = make_inputs(t * world, d, n, f)
    g = make_inputs(t * world, d, 1, f, seed=31, experts=False)["x"]
    r = o.route(full["x"], full["w_router"], k)
    rdh, rdcw, rdwi, rdwo = o.moe_backward(full["x"], full["w_in"], full["w_out"], r["topk_idx"], r["combine_weights"], g)
    parts = [np.load(tmp_path / f"pbwd{i}.npz") for i in range(world)]
    assert np.array_equal(np.concatenate([p_["dh"] for p_ in parts]), rdh)
    assert np.array_equal(np.concatenate([p_["dcw"] for p_ in parts]), rdcw)
    nl = n // world
    for i, p_ in enumerate(parts):
        for e in range(nl):
            if int((r["topk_idx"] == i * nl + e).sum()):
                assert np.array_equal(p_["dwi"][e], rdwi[i * nl + e]), (i, e)
                assert np.array_equal(p_["dwo"][e], rdwo[i * nl + e]), (i, e)
