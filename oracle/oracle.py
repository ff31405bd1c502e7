"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes/numpy front end over the CPU oracle libraries:

* ``liboracle.so``      — the restatement (oracle/moe_oracle.cpp), kind "port";
* ``_ref/libref_moe.so`` — the reference's own primitives (compiled from /root/reference)
  composed per SPEC.md by oracle/ref_compose.cpp, kind "reference".

Only tests/, bench.py's cpu_baseline / ``--impl reference`` leg and __graft_entry__.smoke() may
import this module, and only as the checker. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libref_moe.so")
ROOT_SEED = 20261018

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64 = C.c_int64


class OracleError(RuntimeError):
    """Raised where the reference raises ValidationError / ConfigError."""


def build(ref: bool = False) -> None:
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def available(kind: str) -> bool:
    return os.path.exists(REF_LIB if kind == "reference" else PORT_LIB)


class Oracle:
    """One of the two oracle libraries; same method names for both kinds."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = REF_LIB if kind == "reference" else PORT_LIB
        if not os.path.exists(path):
            if kind == "reference":
                raise FileNotFoundError(f"{path} not built (needs /root/reference; `make -C oracle ref`)")
            build(ref=False)
        self.lib = C.CDLL(path)
        p = "ref_" if kind == "reference" else "orc_"
        self._p = p
        L = self.lib
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "route").argtypes = [_f32p, _f32p, _i64, _i64, _i64, _i64, _f32p, _f32p, _i64p, _f32p, _i64p, _f32p]
        getattr(L, p + "aux_loss").argtypes = [_f32p, _i64p, _i64, _i64, _i64, C.POINTER(C.c_float)]
        getattr(L, p + "z_loss").argtypes = [_f32p, _i64, _i64, C.POINTER(C.c_float)]
        getattr(L, p + "top_k").argtypes = [_f32p, _i64, _i64, _i64p, _f32p]
        getattr(L, p + "moe_forward").argtypes = [_f32p, _i64, _i64, _i64, _i64, _i64, _f32p, _f32p, _i64p, _f32p, _f32p, C.c_int]
        getattr(L, p + "expert_ffn_backward").argtypes = [_f32p, _i64, _i64, _i64, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p]
        getattr(L, p + "moe_backward").argtypes = ([_f32p, _i64, _i64, _i64, _i64, _i64, _f32p, _f32p, _i64p, _f32p, _f32p,
                                                     _f32p, _f32p, _f32p, _f32p] + ([C.c_int] if kind == "port" else []))
        if kind == "port":
            L.orc_split_seed.restype = C.c_uint64
            L.orc_split_seed.argtypes = [C.c_uint64, C.c_uint64]
            L.orc_normals.argtypes = [C.c_uint64, _i64, C.c_float, C.c_float, _f32p]
            L.orc_round_bf16.argtypes = [_f32p, _f32p, _i64]
            L.orc_matmul.argtypes = [_f32p, _f32p, _i64, _i64, _i64, _f32p]
            L.orc_softmax_rows.argtypes = [_f32p, _i64, _i64, _f32p]
            L.orc_plan.argtypes = [_i64p, _i64, _i64, _i64, _i64p, _i64p, _i64p]
            L.orc_expert_ffn.argtypes = [_f32p, _i64, _i64, _i64, _f32p, _f32p, C.c_void_p, _f32p]
            L.orc_fp8_qdq.argtypes = [_f32p, _i64, C.c_float, _f32p]
            L.orc_compute_smoothing.argtypes = [_f32p, _i64, _i64, _i64, _i64, _f32p, _f32p, C.c_float, _f32p]
            L.orc_fold_smoothing.argtypes = [_f32p, _i64, _i64, _i64, _f32p, _f32p, _f32p, _i64]
            L.orc_fp8_encode.argtypes = [_f32p, _i64, _u8p]
            L.orc_router_backward.argtypes = [_f32p, _f32p, _i64, _i64, _i64, _i64, _f32p, _f32p, _i64p, _i64p, _f32p,
                                              C.c_float, C.c_float, _f32p, _f32p]
        else:
            L.ref_gradcheck.argtypes = [C.c_uint64, C.c_int, C.c_double, C.POINTER(C.c_int)]
            L.ref_prng_split.restype = C.c_uint64
            L.ref_prng_split.argtypes = [C.c_uint64, C.c_uint64]
            L.ref_prng_u64.argtypes = [C.c_uint64, C.c_uint64, _i64, np.ctypeslib.ndpointer(np.uint64)]
            L.ref_prng_doubles.argtypes = [C.c_uint64, _i64, np.ctypeslib.ndpointer(np.float64)]
            L.ref_prng_normals.argtypes = [C.c_uint64, _i64, C.c_float, C.c_float, _f32p]
            L.ref_ckpt_resave.argtypes = [C.c_char_p, C.c_char_p]
            L.ref_ckpt_write.argtypes = [C.c_char_p, C.c_char_p, _i64p, _f32p]
            L.ref_moe_backward_full.argtypes = [_f32p, _f32p, _i64, _i64, _i64, _i64, _i64, _f32p, _f32p, _f32p,
                                                C.c_float, C.c_float, _f32p, _f32p, _f32p, _f32p]

    def _call(self, name, *args):
        rc = getattr(self.lib, self._p + name)(*args)
        if rc != 0:
            msg = getattr(self.lib, self._p + "last_error")().decode()
            raise OracleError(msg)

    # ---- SPEC route_tokens / aux_loss / z_loss ----
    def route(self, x: np.ndarray, wr: np.ndarray, k: int):
        x = np.ascontiguousarray(x, np.float32)
        wr = np.ascontiguousarray(wr, np.float32)
        t, d = x.shape
        n = wr.shape[1]
        logits = np.empty((t, n), np.float32)
        probs = np.empty((t, n), np.float32)
        idx = np.empty((t, k), np.int64)
        w = np.empty((t, k), np.float32)
        counts = np.empty(n, np.int64)
        aggp = np.empty(n, np.float32)
        self._call("route", x, wr, t, d, n, k, logits, probs, idx, w, counts, aggp)
        return dict(logits=logits, probs=probs, topk_idx=idx, combine_weights=w, counts=counts,
                    agg_prob=aggp, B=t, K=k)

    def aux_loss(self, probs, counts, k: int) -> float:
        probs = np.ascontiguousarray(probs, np.float32)
        out = C.c_float()
        self._call("aux_loss", probs, np.ascontiguousarray(counts, np.int64), probs.shape[0], probs.shape[1], k, C.byref(out))
        return out.value

    def z_loss(self, logits) -> float:
        logits = np.ascontiguousarray(logits, np.float32)
        out = C.c_float()
        self._call("z_loss", logits, logits.shape[0], logits.shape[1], C.byref(out))
        return out.value

    def top_k(self, x, k: int):
        x = np.ascontiguousarray(x, np.float32)
        idx = np.empty(max(k, 1), np.int64)
        val = np.empty(max(k, 1), np.float32)
        self._call("top_k", x, x.size, k, idx, val)
        return idx[:k], val[:k]

    def moe_forward(self, x, w_in, w_out, idx, w, jobs: int = 1):
        x = np.ascontiguousarray(x, np.float32)
        t, d = x.shape
        n, _, f2 = w_in.shape
        k = idx.shape[1]
        out = np.empty((t, d), np.float32)
        self._call("moe_forward", x, t, d, n, k, f2 // 2, np.ascontiguousarray(w_in, np.float32),
                   np.ascontiguousarray(w_out, np.float32), np.ascontiguousarray(idx, np.int64),
                   np.ascontiguousarray(w, np.float32), out, jobs)
        return out

    def expert_ffn_backward(self, xe, w_in_e, w_out_e, dy):
        xe = np.ascontiguousarray(xe, np.float32)
        m, d = xe.shape
        f = w_out_e.shape[0]
        dx = np.empty((m, d), np.float32)
        dwi = np.empty((d, 2 * f), np.float32)
        dwo = np.empty((f, d), np.float32)
        self._call("expert_ffn_backward", xe, m, d, f, np.ascontiguousarray(w_in_e, np.float32),
                   np.ascontiguousarray(w_out_e, np.float32), np.ascontiguousarray(dy, np.float32), dx, dwi, dwo)
        return dx, dwi, dwo

    def moe_backward(self, x, w_in, w_out, idx, w, d_out, jobs: int = 1):
        """Layer backward: returns (d_hidden [T x d], d_combine_w [T x K], dw_in [N][d][2f], dw_out [N][f][d])."""
        x = np.ascontiguousarray(x, np.float32)
        t, d = x.shape
        n, _, f2 = w_in.shape
        k = idx.shape[1]
        dh = np.empty((t, d), np.float32)
        dcw = np.empty((t, k), np.float32)
        dwi = np.empty((n, d, f2), np.float32)
        dwo = np.empty((n, f2 // 2, d), np.float32)
        args = [x, t, d, n, k, f2 // 2, np.ascontiguousarray(w_in, np.float32), np.ascontiguousarray(w_out, np.float32),
                np.ascontiguousarray(idx, np.int64), np.ascontiguousarray(w, np.float32),
                np.ascontiguousarray(d_out, np.float32), dh, dcw, dwi, dwo]
        if self.kind == "port":
            args.append(jobs)
        self._call("moe_backward", *args)
        return dh, dcw, dwi, dwo

    def moe_backward_full(self, x, wr, w_in, w_out, d_out, g_aux, g_z, k, jobs: int = 1):
        """Layer + router backward: (d_hidden, dW_r, dW_in, dW_out). "reference": the Tape over the
        reference ops; "port": orc_moe_backward + orc_router_backward (analytic router part)."""
        x = np.ascontiguousarray(x, np.float32)
        wr = np.ascontiguousarray(wr, np.float32)
        t, d = x.shape
        n, _, f2 = w_in.shape
        dh = np.empty((t, d), np.float32)
        dwr = np.empty((d, n), np.float32)
        dwi = np.empty((n, d, f2), np.float32)
        dwo = np.empty((n, f2 // 2, d), np.float32)
        d_out = np.ascontiguousarray(d_out, np.float32)
        if self.kind == "reference":
            self._call("moe_backward_full", x, wr, t, d, n, k, f2 // 2, np.ascontiguousarray(w_in, np.float32),
                       np.ascontiguousarray(w_out, np.float32), d_out, g_aux, g_z, dh, dwr, dwi, dwo)
            return dh, dwr, dwi, dwo
        r = self.route(x, wr, k)
        dh, dcw, dwi, dwo = self.moe_backward(x, w_in, w_out, r["topk_idx"], r["combine_weights"], d_out, jobs=jobs)
        self._call("router_backward", x, wr, t, d, n, k, r["logits"], r["probs"], r["topk_idx"], r["counts"], dcw,
                   g_aux, g_z, dh, dwr)
        return dh, dwr, dwi, dwo

    # ---- port-only helpers ----
    def expert_ffn(self, xe, w_in_e, w_out_e):
        xe = np.ascontiguousarray(xe, np.float32)
        m, d = xe.shape
        f = w_out_e.shape[0]
        a = np.empty((m, f), np.float32)
        y = np.empty((m, d), np.float32)
        self._call("expert_ffn", xe, m, d, f, np.ascontiguousarray(w_in_e, np.float32),
                   np.ascontiguousarray(w_out_e, np.float32), a.ctypes.data, y)
        return a, y

    def plan(self, idx, n: int):
        idx = np.ascontiguousarray(idx, np.int64)
        t, k = idx.shape
        offsets = np.empty(n + 1, np.int64)
        perm = np.empty(t * k, np.int64)
        inv = np.empty(t * k, np.int64)
        self.lib.orc_plan(idx, t, n, k, offsets, perm, inv)
        return offsets, perm, inv

    def matmul(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty((a.shape[0], b.shape[1]), np.float32)
        self._call("matmul", a, b, a.shape[0], a.shape[1], b.shape[1], out)
        return out

    def softmax_rows(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self._call("softmax_rows", x, x.shape[0], x.shape[1], out)
        return out

    def fp8_qdq(self, x, scale: float):
        x = np.ascontiguousarray(x, np.float32).ravel()
        out = np.empty_like(x)
        self._call("fp8_qdq", x, x.size, scale, out)
        return out

    def compute_smoothing(self, x, w_in, wr, alpha):
        x = np.ascontiguousarray(x, np.float32)
        t, d = x.shape
        n, _, f2 = w_in.shape
        s = np.empty(d, np.float32)
        self.lib.orc_compute_smoothing(x, t, d, n, f2 // 2, np.ascontiguousarray(w_in, np.float32),
                                       np.ascontiguousarray(wr, np.float32), alpha, s)
        return s

    def fold_smoothing(self, s, w_in, wr, x):
        """Returns folded copies (w_in', wr', x / s)."""
        w_in = np.array(w_in, np.float32, copy=True)
        wr = np.array(wr, np.float32, copy=True)
        x = np.array(x, np.float32, copy=True)
        n, d, f2 = w_in.shape
        self.lib.orc_fold_smoothing(np.ascontiguousarray(s, np.float32), d, n, f2 // 2, w_in, wr, x, x.shape[0])
        return w_in, wr, x

    def fp8_encode(self, q):
        q = np.ascontiguousarray(q, np.float32).ravel()
        out = np.empty(q.size, np.uint8)
        self._call("fp8_encode", q, q.size, out)
        return out

    def split_seed(self, root: int, stream: int) -> int:
        if self.kind == "reference":
            return self.lib.ref_prng_split(root, stream)
        return self.lib.orc_split_seed(root, stream)

    def normals(self, seed: int, n: int, stddev: float, mean: float = 0.0):
        out = np.empty(n, np.float32)
        if self.kind == "reference":
            self.lib.ref_prng_normals(seed, n, mean, stddev, out)
        else:
            self.lib.orc_normals(seed, n, mean, stddev, out)
        return out

    # ---- the reference Prng itself (kind "reference" only) ----
    def prng_u64(self, seed: int, n: int, counter: int = 0):
        out = np.empty(n, np.uint64)
        self.lib.ref_prng_u64(seed, counter, n, out)
        return out

    def prng_doubles(self, seed: int, n: int):
        out = np.empty(n, np.float64)
        self.lib.ref_prng_doubles(seed, n, out)
        return out

    def round_bf16(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.lib.orc_round_bf16(x.ravel(), out.ravel(), x.size)
        return out

    # ---- SPEC balance_calibration, restated over route() ----
    def balance_calibration(self, base, pool, wr, k: int, tau: int):
        """Counts of the routed base set, then pool tokens in order: a token is taken iff one of
        its top-k experts is still below tau; stop once every expert reaches tau. Returns
        (selected pool indices, final counts); raises OracleError naming the expert when the pool
        runs out first. Pure-Python loop: small cases only."""
        if tau < 1:
            raise OracleError("balance_calibration: tau must be >= 1")
        n = wr.shape[1]
        cnt = np.zeros(n, np.int64)
        if base is not None and len(base):
            cnt += self.route(base, wr, k)["counts"]
        sel = []
        if pool is not None and len(pool) and (cnt < tau).any():
            idx = self.route(pool, wr, k)["topk_idx"]
            for j in range(idx.shape[0]):
                if not (cnt < tau).any():
                    break
                if (cnt[idx[j]] < tau).any():
                    cnt[idx[j]] += 1
                    sel.append(j)
        low = np.nonzero(cnt < tau)[0]
        if len(low):
            e = int(low[0])
            raise OracleError(f"balance_calibration: token pool exhausted with expert {e} at {cnt[e]} < tau={tau}")
        return np.array(sel, np.int64), cnt

    # ---- reference checkpoint code (kind "reference" only) ----
    def ckpt_resave(self, src: str, dst: str) -> None:
        self._call("ckpt_resave", src.encode(), dst.encode())

    def ckpt_write(self, path: str, tensors: dict) -> None:
        names = "\n".join(tensors)
        shapes, vals = [], []
        for a in tensors.values():
            a = np.ascontiguousarray(a, np.float32)
            shapes += [a.ndim] + list(a.shape)
            vals.append(a.ravel())
        self._call("ckpt_write", path.encode(), names.encode(), np.array(shapes, np.int64),
                   np.ascontiguousarray(np.concatenate(vals), np.float32))

    def gradcheck(self, seed=20260809, cases=100, tol=1e-4):
        n = C.c_int()
        fails = self.lib.ref_gradcheck(seed, cases, tol, C.byref(n))
        return fails, n.value


def make_inputs(t: int, d: int, n: int, f: int, seed: int = ROOT_SEED, bf16: bool = True,
                skew: float | None = None, experts: bool = True):
    """Synthetic layer inputs per SURVEY.md §8(d), drawn with the reference Prng streams.

    x = split(1) N(0,1); W_r = split(2) N(0,1/sqrt d); W_in[e] = split(16+e) N(0,1/sqrt d);
    W_out[e] = split(16+N+e) N(0,1/sqrt f). x and the expert weights are rounded to bf16 when
    ``bf16`` (the device path's storage type); the router stays fp32. ``skew`` = gamma of the C5
    mean-shift construction (x += 1; W_r[:, i] += gamma*ln(1/(i+1)^1.2)/d).
    """
    o = Oracle("port")
    sd = float(np.float32(1.0 / np.sqrt(d)))
    sf = float(np.float32(1.0 / np.sqrt(f)))
    x = o.normals(o.split_seed(seed, 1), t * d, 1.0).reshape(t, d)
    wr = o.normals(o.split_seed(seed, 2), d * n, sd).reshape(d, n)
    if skew is not None:
        x = (x + np.float32(1.0)).astype(np.float32)
        beta = np.array([skew * np.log(1.0 / (i + 1) ** 1.2) for i in range(n)], np.float64)
        wr = (wr + (beta / d).astype(np.float32)[None, :]).astype(np.float32)
    out = dict(x=o.round_bf16(x) if bf16 else x, w_router=wr)
    if experts:
        w_in = np.empty((n, d, 2 * f), np.float32)
        w_out = np.empty((n, f, d), np.float32)
        for e in range(n):
            w_in[e] = o.normals(o.split_seed(seed, 16 + e), d * 2 * f, sd).reshape(d, 2 * f)
            w_out[e] = o.normals(o.split_seed(seed, 16 + n + e), f * d, sf).reshape(f, d)
        if bf16:
            w_in = o.round_bf16(w_in)
            w_out = o.round_bf16(w_out)
        out.update(w_in=w_in, w_out=w_out)
    return out


def router_fp8_sim(o: Oracle, x, wr, k: int, s_x: float):
    """route_tokens of the quantized model (the router GEMM runs through fp8_qdq too):
    x_hat = qdq(x, s_x) with the per-tensor activation scale, W_r_hat[:, i] = qdq(W_r[:, i], s_w[i])
    with s_w[i] = absmax of expert column i / 448 (1 for an all-zero column); then the reference
    route on those dequantised fp32 values. Returns (decision, s_w [N])."""
    x = np.ascontiguousarray(x, np.float32)
    wr = np.ascontiguousarray(wr, np.float32)
    t, d = x.shape
    n = wr.shape[1]
    m = np.abs(wr).max(0)
    s_w = np.where(m > 0, m / np.float32(448.0), np.float32(1.0)).astype(np.float32)
    xq = o.fp8_qdq(x, float(s_x)).reshape(t, d)
    wq = np.empty_like(wr)
    for c in range(n):
        wq[:, c] = o.fp8_qdq(wr[:, c], float(s_w[c]))
    return o.route(xq, wq, k), s_w


def moe_forward_fp8_sim(o: Oracle, x, w_in, w_out, idx, w, s_in, s_mid, ws_in=None, ws_out=None):
    """Expert-aware FP8 layer simulated with the oracle's E4M3 qdq:
    per expert e, X_e -> qdq(X_e, s_in[e]); every output channel of W_in[e] / W_out[e] -> qdq with
    scale = channel absmax / 448 (per-output-channel weight scales); GEMMs in
    float64; A = silu(G) * U -> qdq(A, s_mid[e]); Y = A_q W_out_q; out = sum_k w * Y in slot order.
    Returns (out float64 [T x d], ws_in [N x 2f] (reference column order), ws_out [N x d])."""
    t, d = x.shape
    n, _, f2 = w_in.shape
    f = f2 // 2
    k = idx.shape[1]
    if ws_in is None:
        ws_in = np.empty((n, f2), np.float32)
        ws_out = np.empty((n, d), np.float32)
        for e in range(n):
            m = np.abs(w_in[e]).max(0)
            ws_in[e] = np.where(m > 0, m / np.float32(448.0), np.float32(1.0))
            m = np.abs(w_out[e]).max(0)
            ws_out[e] = np.where(m > 0, m / np.float32(448.0), np.float32(1.0))
    out = np.zeros((t, d), np.float64)
    for e in range(n):
        rows, slots = np.nonzero(idx == e)
        if len(rows) == 0:
            continue
        xq = o.fp8_qdq(x[rows], float(s_in[e])).reshape(len(rows), d)
        wq = np.empty_like(w_in[e])
        for c in range(f2):
            wq[:, c] = o.fp8_qdq(w_in[e][:, c], float(ws_in[e][c]))
        h = xq.astype(np.float64) @ wq.astype(np.float64)
        g, u = h[:, :f], h[:, f:]
        a = (g / (1.0 + np.exp(-g)) * u).astype(np.float32)
        aq = o.fp8_qdq(a, float(s_mid[e])).reshape(a.shape)
        woq = np.empty_like(w_out[e])
        for c in range(d):
            woq[:, c] = o.fp8_qdq(w_out[e][:, c], float(ws_out[e][c]))
        y = aq.astype(np.float64) @ woq.astype(np.float64)
        out[rows] += w[rows, slots][:, None].astype(np.float64) * y
    return out, ws_in, ws_out
