"""Host-side mirror of the reference's MoE-layer operator interface.

Same operation names, argument meaning and error behaviour as the SPEC ops, backed by the
sm_100a kernels through the C ABI (include/compass_moe.h):

* ``route_tokens(hidden) -> RouterDecision``
* ``moe_forward(hidden, decision) -> Tensor[B x d]``
* ``aux_loss(decision)`` / ``z_loss(decision)``        SPEC.md:165-182 (computed on device)
* ``calibrate`` / ``quantize_fp8``                     SPEC.md:532-570 (expert-aware FP8)

Device tensors are torch CUDA tensors (torch is used for device memory and streams only).
Errors: ``MoEConfigError`` for CL_ERR_CONFIG, ``MoEError`` for CL_ERR_RUN (ValidationError).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import MoEConfigError, MoEError  # noqa: F401  (re-exported)


@dataclass
class MoEConfig:
    d_model: int
    n_experts: int
    top_k: int
    d_ff: int
    max_tokens: int
    device: int = 0
    gemm_ctas: int = 0  # 0 auto (2-CTA), 1 or 2
    ep_size: int = 1
    ep_rank: int = 0

    def to_c(self) -> _lib.Config:
        return _lib.Config(self.d_model, self.n_experts, self.top_k, self.d_ff, self.max_tokens, self.device,
                           self.gemm_ctas, self.ep_size, self.ep_rank)


@dataclass
class RouterDecision:
    """logits z, probs, topk_idx, combine_weights, counts c, agg_prob p, B, K."""
    logits: torch.Tensor
    probs: torch.Tensor
    topk_idx: torch.Tensor
    combine_weights: torch.Tensor
    counts: torch.Tensor
    agg_prob: torch.Tensor
    aux: torch.Tensor
    z: torch.Tensor
    B: int
    K: int


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class MoELayer:
    """One MoE layer (router + N gated experts) resident on one B200."""

    def __init__(self, cfg: MoEConfig, w_router=None, w_in=None, w_out=None, seed: int | None = None,
                 checkpoint: str | None = None, prefix: str = ""):
        self.cfg = cfg
        self.L = _lib.lib()
        self.h = C.c_void_p()
        self.device = torch.device("cuda", cfg.device)
        c = cfg.to_c()
        if checkpoint is not None:
            rc = self.L.cl_moe_create_from_checkpoint(C.byref(c), checkpoint.encode(), prefix.encode(), C.byref(self.h))
        elif seed is not None:
            rc = self.L.cl_moe_create_synthetic(C.byref(c), seed, C.byref(self.h))
        else:
            wr = np.ascontiguousarray(w_router, np.float32)
            wi = np.ascontiguousarray(w_in, np.float32)
            wo = np.ascontiguousarray(w_out, np.float32)
            rc = self.L.cl_moe_create(C.byref(c), wr.ctypes.data, wi.ctypes.data, wo.ctypes.data, C.byref(self.h))
        if rc != _lib.CL_OK:
            cls = MoEConfigError if rc == _lib.CL_ERR_CONFIG else MoEError
            raise cls(f"cl_moe_create failed with status {rc}: {self.L.cl_moe_last_error(None).decode()}")

    def close(self):
        if self.h:
            self.L.cl_moe_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        _lib.check(rc, self.h, what)

    # ---------------------------------------------------------------- SPEC ops
    def route_tokens(self, hidden: torch.Tensor) -> RouterDecision:
        """bf16 hidden, or fp32 hidden (the reference's Tensor dtype): fp32 is routed on its own
        values, bit-exact with the reference's route_tokens on the same tensor."""
        t = hidden.shape[0]
        dec = self._new_decision(t)
        cd = self._decision_struct(dec)
        if hidden.dtype == torch.float32:
            rc = self.L.cl_moe_route_tokens_f32(self.h, _ptr(self._f32(hidden)), t, C.byref(cd), _stream(self.device))
        else:
            rc = self.L.cl_moe_route_tokens(self.h, _ptr(self._bf16(hidden)), t, C.byref(cd), _stream(self.device))
        self._check(rc, "route_tokens")
        return dec

    def moe_forward(self, hidden: torch.Tensor, decision: RouterDecision) -> torch.Tensor:
        hidden = self._bf16(hidden)
        out = torch.empty_like(hidden)
        idx = decision.topk_idx.to(torch.int32).contiguous()
        w = decision.combine_weights.to(torch.float32).contiguous()
        self._check(self.L.cl_moe_moe_forward(self.h, _ptr(hidden), hidden.shape[0], _ptr(idx), _ptr(w), _ptr(out),
                                              _stream(self.device)), "moe_forward")
        return out

    def forward(self, hidden: torch.Tensor, want_decision: bool = False):
        """route_tokens + moe_forward fused on device. Returns out (and the decision).
        fp32 hidden: routed on the fp32 values, experts on their bf16 rounding, fp32 out."""
        f32 = hidden.dtype == torch.float32
        hidden = self._f32(hidden) if f32 else self._bf16(hidden)
        out = torch.empty_like(hidden)
        dec = None
        cd = None
        if want_decision:
            dec = self._new_decision(hidden.shape[0])
            cd = C.byref(self._decision_struct(dec))
        fn = self.L.cl_moe_forward_f32 if f32 else self.L.cl_moe_forward
        self._check(fn(self.h, _ptr(hidden), hidden.shape[0], _ptr(out), cd, _stream(self.device)), "forward")
        return (out, dec) if want_decision else out

    def forward_graph(self, hidden: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """forward() replayed from a CUDA graph captured per (hidden, out, T, precision)."""
        hidden = self._bf16(hidden)
        out = torch.empty_like(hidden) if out is None else out
        self._check(self.L.cl_moe_forward_graph(self.h, _ptr(hidden), hidden.shape[0], _ptr(out), _stream(self.device)),
                    "forward_graph")
        return out

    def forward_host(self, x: np.ndarray, io_dtype: str = "bf16") -> np.ndarray:
        """Reference-facing call on HOST buffers (H2D + layer + D2H, synchronous).

        ``x`` is float32 [T x d] (io_dtype "f32") or a uint16 array of bf16 bits ("bf16")."""
        t = x.shape[0]
        if io_dtype == "f32":
            x = np.ascontiguousarray(x, np.float32)
            out = np.empty_like(x)
            code = _lib.CL_MOE_IO_F32
        else:
            x = np.ascontiguousarray(x, np.uint16)
            out = np.empty_like(x)
            code = _lib.CL_MOE_IO_BF16
        self._check(self.L.cl_moe_forward_host(self.h, x.ctypes.data, t, out.ctypes.data, code), "forward_host")
        return out

    def forward_host_ptr(self, x_ptr: int, t: int, out_ptr: int, io_dtype: int = _lib.CL_MOE_IO_BF16) -> None:
        self._check(self.L.cl_moe_forward_host(self.h, C.c_void_p(x_ptr), t, C.c_void_p(out_ptr), io_dtype),
                    "forward_host")

    def forward_host_async(self, x_ptr: int, t: int, out_ptr: int, io_dtype: int = _lib.CL_MOE_IO_BF16) -> None:
        """Pipelined host-buffer call (pinned buffers); completes at host_wait()."""
        self._check(self.L.cl_moe_forward_host_async(self.h, C.c_void_p(x_ptr), t, C.c_void_p(out_ptr), io_dtype),
                    "forward_host_async")

    def host_wait(self) -> None:
        self._check(self.L.cl_moe_host_wait(self.h), "host_wait")

    @staticmethod
    def aux_loss(decision: RouterDecision) -> float:
        return float(decision.aux.item())

    @staticmethod
    def z_loss(decision: RouterDecision) -> float:
        return float(decision.z.item())

    def sync(self):
        self._check(self.L.cl_moe_sync(self.h, _stream(self.device)), "sync")

    # ---------------------------------------------------------------- FP8 (SPEC expert-quantizer)
    def calibrate(self, hidden: torch.Tensor, reset: bool = True):
        self._check(self.L.cl_moe_calibrate(self.h, _ptr(self._bf16(hidden)), hidden.shape[0], int(reset),
                                            _stream(self.device)), "calibrate")

    def quantize_fp8(self, act_scale_in=None, act_scale_mid=None, router_act_scale=None):
        """quantize_model. Explicit scales: act_scale_in [N], act_scale_mid
        [N_local], router_act_scale (the router's per-tensor activation scale; else calibration)."""
        if router_act_scale is not None:
            self.set_router_fp8(True, router_act_scale)
        if act_scale_in is None:
            rc = self.L.cl_moe_quantize_fp8(self.h, None, None)
        else:
            a = np.ascontiguousarray(act_scale_in, np.float32)  # [N]: every expert (EP: global table)
            b = np.ascontiguousarray(act_scale_mid, np.float32)  # [N_local]
            if a.size != self.cfg.n_experts or b.size != self.cfg.n_experts // self.cfg.ep_size:
                raise MoEConfigError("act_scale_in needs n_experts entries, act_scale_mid n_experts/ep_size")
            rc = self.L.cl_moe_quantize_fp8(self.h, a.ctypes.data, b.ctypes.data)
        self._check(rc, "quantize_fp8")

    def set_router_fp8(self, enable: bool = True, act_scale: float = 0.0):
        """Router GEMM through fp8_qdq in FP8 mode (default) or fp32 gating (False).
        act_scale > 0 fixes the router's activation scale (else: calibration max / 448)."""
        self._check(self.L.cl_moe_set_router_fp8(self.h, int(enable), float(act_scale)), "set_router_fp8")

    def router_stats(self):
        """(certified routing calls so far, tokens recomputed exactly in the last one)."""
        a, b = C.c_int64(), C.c_int64()
        self._check(self.L.cl_moe_router_stats(self.h, C.byref(a), C.byref(b)), "router_stats")
        return a.value, b.value

    def router_variant(self):
        """(K1 kernel of the last routing call — 0..6, see compass_moe.h —, DMMA device check passed)."""
        a, b = C.c_int32(), C.c_int32()
        self._check(self.L.cl_moe_router_variant(self.h, C.byref(a), C.byref(b)), "router_variant")
        return a.value, bool(b.value)

    def router_weights(self) -> np.ndarray:
        """Host copy of W_r [d x N] (fp32) as the layer holds it."""
        w = np.empty((self.cfg.d_model, self.cfg.n_experts), np.float32)
        self._check(self.L.cl_moe_get_weights(self.h, w.ctypes.data, 0, None, None), "get_weights")
        return w

    def expert_weights(self, e: int):
        """Host copies of local expert e's (W_in [d x 2f], W_out [f x d]) in the reference layouts."""
        d, f = self.cfg.d_model, self.cfg.d_ff
        wi = np.empty((d, 2 * f), np.float32)
        wo = np.empty((f, d), np.float32)
        self._check(self.L.cl_moe_get_weights(self.h, None, e, wi.ctypes.data, wo.ctypes.data), "get_weights")
        return wi, wo

    def save_fp8_scheme(self, path: str) -> None:
        """QuantScheme file: JSON manifest at `path`, fp32 scale arrays in `path`.bin."""
        self._check(self.L.cl_moe_save_fp8_scheme(self.h, path.encode()), "save_fp8_scheme")

    def load_fp8_scheme(self, path: str) -> None:
        """Applies a saved scheme (fold, scales, weight quantization) and switches to FP8."""
        self._check(self.L.cl_moe_load_fp8_scheme(self.h, path.encode()), "load_fp8_scheme")

    def router_fp8_scales(self):
        """(enabled, activation scale, weight scales [N]) of the router under the FP8 scheme."""
        en = C.c_int32()
        a = C.c_float()
        w = np.empty(self.cfg.n_experts, np.float32)
        self._check(self.L.cl_moe_get_router_fp8(self.h, C.byref(en), C.byref(a), w.ctypes.data), "router_fp8_scales")
        return bool(en.value), a.value, w

    def calibration_stats(self):
        """collect_calibration statistics: dict(counts [N], x_max [N_local], mid_max [N_local], ch_max [d])."""
        nl = self.cfg.n_experts // self.cfg.ep_size
        out = dict(counts=np.zeros(self.cfg.n_experts, np.int64), x_max=np.zeros(nl, np.float32),
                   mid_max=np.zeros(nl, np.float32), ch_max=np.zeros(self.cfg.d_model, np.float32))
        self._check(self.L.cl_moe_calibration_stats(self.h, *(v.ctypes.data for v in out.values())),
                    "calibration_stats")
        return out

    def save_checkpoint(self, path: str, prefix: str = "") -> None:
        self._check(self.L.cl_moe_save_checkpoint(self.h, path.encode(), prefix.encode()), "save_checkpoint")

    def balance_calibration(self, base, pool, tau: int):
        """SPEC balance_calibration: (selected pool row indices, final counts)."""
        base = None if base is None else self._bf16(base)
        pool = None if pool is None else self._bf16(pool)
        p = 0 if pool is None else pool.shape[0]
        sel = np.empty(max(p, 1), np.int64)
        ns = C.c_int64()
        fc = np.empty(self.cfg.n_experts, np.int64)
        self._check(self.L.cl_moe_balance_calibration(self.h, _ptr(base), 0 if base is None else base.shape[0],
                                                      _ptr(pool), p, tau, sel.ctypes.data, C.byref(ns), fc.ctypes.data,
                                                      _stream(self.device)), "balance_calibration")
        return sel[:ns.value], fc

    def compute_smoothing(self, alpha: float = 0.5) -> np.ndarray:
        s = np.empty(self.cfg.d_model, np.float32)
        self._check(self.L.cl_moe_compute_smoothing(self.h, alpha, s.ctypes.data), "compute_smoothing")
        return s

    def fold_smoothing(self, s) -> None:
        s = np.ascontiguousarray(s, np.float32)
        self._check(self.L.cl_moe_fold_smoothing(self.h, s.ctypes.data), "fold_smoothing")

    def set_precision(self, precision: str):
        code = _lib.CL_MOE_FP8_E4M3 if precision == "fp8" else _lib.CL_MOE_BF16
        self._check(self.L.cl_moe_set_precision(self.h, code), "set_precision")

    def fp8_scales(self):
        nl = self.cfg.n_experts // self.cfg.ep_size
        d, f = self.cfg.d_model, self.cfg.d_ff
        a = np.empty(nl, np.float32)
        b = np.empty(nl, np.float32)
        wi = np.empty((nl, 2 * f), np.float32)
        wo = np.empty((nl, d), np.float32)
        self._check(self.L.cl_moe_get_fp8_scales(self.h, a.ctypes.data, b.ctypes.data, wi.ctypes.data, wo.ctypes.data),
                    "fp8_scales")
        return a, b, wi, wo

    # ---------------------------------------------------------------- training (expert-FFN backward)
    def forward_train(self, hidden: torch.Tensor, want_decision: bool = False):
        hidden = self._bf16(hidden)
        out = torch.empty_like(hidden)
        dec, cd = None, None
        if want_decision:
            dec = self._new_decision(hidden.shape[0])
            cd = C.byref(self._decision_struct(dec))
        self._check(self.L.cl_moe_forward_train(self.h, _ptr(hidden), hidden.shape[0], _ptr(out), cd,
                                                _stream(self.device)), "forward_train")
        return (out, dec) if want_decision else out

    def backward(self, d_out: torch.Tensor):
        """Expert-FFN backward of the last forward_train: (d_hidden, d_combine_w, dW_in, dW_out)."""
        d_out = self._bf16(d_out)
        t = d_out.shape[0]
        nl = self.cfg.n_experts // self.cfg.ep_size
        d, f, k = self.cfg.d_model, self.cfg.d_ff, self.cfg.top_k
        dh = torch.empty_like(d_out)
        dcw = torch.empty(t, k, dtype=torch.float32, device=self.device)
        dwi = torch.empty(nl, d, 2 * f, dtype=torch.float32, device=self.device)
        dwo = torch.empty(nl, f, d, dtype=torch.float32, device=self.device)
        self._check(self.L.cl_moe_backward(self.h, _ptr(d_out), _ptr(dh), _ptr(dcw), _ptr(dwi), _ptr(dwo),
                                           _stream(self.device)), "backward")
        return dh, dcw, dwi, dwo

    def backward_full(self, d_out: torch.Tensor, g_aux: float = 0.0, g_z: float = 0.0):
        """Layer + router backward of the last forward_train: (d_hidden, dW_r, dW_in, dW_out)."""
        d_out = self._bf16(d_out)
        nl = self.cfg.n_experts // self.cfg.ep_size
        d, f, n = self.cfg.d_model, self.cfg.d_ff, self.cfg.n_experts
        dh = torch.empty_like(d_out)
        dwr = torch.empty(d, n, dtype=torch.float32, device=self.device)
        dwi = torch.empty(nl, d, 2 * f, dtype=torch.float32, device=self.device)
        dwo = torch.empty(nl, f, d, dtype=torch.float32, device=self.device)
        self._check(self.L.cl_moe_backward_full(self.h, _ptr(d_out), g_aux, g_z, _ptr(dh), _ptr(dwr), _ptr(dwi),
                                                _ptr(dwo), None, _stream(self.device)), "backward_full")
        return dh, dwr, dwi, dwo

    def _new_decision(self, t: int) -> "RouterDecision":
        n, k, dev = self.cfg.n_experts, self.cfg.top_k, self.device
        return RouterDecision(
            logits=torch.empty(t, n, dtype=torch.float32, device=dev),
            probs=torch.empty(t, n, dtype=torch.float32, device=dev),
            topk_idx=torch.empty(t, k, dtype=torch.int32, device=dev),
            combine_weights=torch.empty(t, k, dtype=torch.float32, device=dev),
            counts=torch.empty(n, dtype=torch.int64, device=dev),
            agg_prob=torch.empty(n, dtype=torch.float32, device=dev),
            aux=torch.empty(1, dtype=torch.float32, device=dev),
            z=torch.empty(1, dtype=torch.float32, device=dev), B=t, K=k)

    # ---------------------------------------------------------------- expert parallelism
    @staticmethod
    def ep_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        rc = _lib.lib().cl_moe_ep_unique_id(buf)
        if rc != _lib.CL_OK:
            raise MoEError("cl_moe_ep_unique_id failed")
        return bytes(buf)

    def ep_init(self, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self.L.cl_moe_ep_init(self.h, buf), "ep_init")

    def ep_peer_init(self):
        """Collective: switch to the NVLink peer-memory transport (cl_moe_ep_peer_init)."""
        self._check(self.L.cl_moe_ep_peer_init(self.h), "ep_peer_init")

    def ep_last_counts(self) -> np.ndarray:
        """R x N routing counts all-gathered by the last expert-parallel forward (row = source)."""
        c = np.empty((self.cfg.ep_size, self.cfg.n_experts), np.int64)
        self._check(self.L.cl_moe_ep_last_counts(self.h, c.ctypes.data), "ep_last_counts")
        return c

    def ep_forward(self, hidden: torch.Tensor) -> torch.Tensor:
        hidden = self._bf16(hidden)
        out = torch.empty_like(hidden)
        self._check(self.L.cl_moe_ep_forward(self.h, _ptr(hidden), hidden.shape[0], _ptr(out), None,
                                             _stream(self.device)), "ep_forward")
        return out

    # ---------------------------------------------------------------- per-stage timing
    STAGES = ("router", "plan", "dispatch", "gemm1", "gemm2", "combine",
              "combine_bwd", "dgrad1_swiglu_bwd", "dgrad2", "dispatch_bwd", "transposes", "wgrad_out", "wgrad_in")

    def profile(self, enable: bool = True):
        self._check(self.L.cl_moe_profile(self.h, int(enable)), "profile")

    def profile_read(self):
        """Summed per-stage ms since the last read, and (forward calls, backward calls)."""
        ms = (C.c_double * 16)()
        calls = (C.c_int64 * 2)()
        self._check(self.L.cl_moe_profile_read(self.h, ms, calls), "profile_read")
        return {k: ms[i] for i, k in enumerate(self.STAGES)}, (calls[0], calls[1])

    # ---------------------------------------------------------------- stage access (tests)
    def stage(self, name: str, shape, dtype) -> torch.Tensor:
        out = torch.empty(shape, dtype=dtype, device=self.device)
        nbytes = out.numel() * out.element_size()
        self._check(self.L.cl_moe_copy_stage(self.h, _lib.STAGE[name], _ptr(out), nbytes, _stream(self.device)),
                    "copy_stage")
        return out

    def synthetic_tokens(self, t: int, seed: int, shift: float = 0.0) -> torch.Tensor:
        x = torch.empty(t, self.cfg.d_model, dtype=torch.bfloat16, device=self.device)
        self._check(self.L.cl_moe_synthetic_tokens_shifted(self.h, seed, t, shift, _ptr(x), _stream(self.device)),
                    "synthetic_tokens")
        return x

    def synthetic_skew(self, gamma: float):
        self._check(self.L.cl_moe_synthetic_skew(self.h, gamma), "synthetic_skew")

    # ---------------------------------------------------------------- helpers
    def _bf16(self, x: torch.Tensor) -> torch.Tensor:
        if x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous():
            raise MoEConfigError("hidden must be a contiguous bf16 CUDA tensor [B x d]")
        if x.shape[1] != self.cfg.d_model:
            raise MoEConfigError(f"hidden has {x.shape[1]} columns, expected d_model={self.cfg.d_model}")
        return x

    def _f32(self, x: torch.Tensor) -> torch.Tensor:
        if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
            raise MoEConfigError("hidden must be a contiguous fp32 CUDA tensor [B x d]")
        if x.shape[1] != self.cfg.d_model:
            raise MoEConfigError(f"hidden has {x.shape[1]} columns, expected d_model={self.cfg.d_model}")
        return x

    @staticmethod
    def _decision_struct(dec: RouterDecision) -> _lib.Decision:
        return _lib.Decision(dec.logits.data_ptr(), dec.probs.data_ptr(), dec.topk_idx.data_ptr(),
                             dec.combine_weights.data_ptr(), dec.counts.data_ptr(), dec.agg_prob.data_ptr(),
                             dec.aux.data_ptr(), dec.z.data_ptr())


def ep_layout(counts: np.ndarray, rank: int):
    """Receive layout of `rank` from the all-gathered [R x N] count matrix (pure host, no GPU):
    returns (local_offsets [N/R+1], recv_piece [N/R x R], total)."""
    counts = np.ascontiguousarray(counts, np.int64)
    r, n = counts.shape
    nl = n // r
    loc = np.empty(nl + 1, np.int64)
    piece = np.empty(nl * r, np.int64)
    tot = C.c_int64()
    rc = _lib.lib().cl_moe_ep_layout(counts.ctypes.data, r, n, rank, loc.ctypes.data, piece.ctypes.data, C.byref(tot))
    if rc != _lib.CL_OK:
        raise MoEConfigError("ep_layout: bad arguments")
    return loc, piece.reshape(nl, r), tot.value


def ep_peer_layout(counts: np.ndarray, rank: int):
    """Peer-transport layout of `rank` (pure host): (dispatch_row [N], return_row [N/R x R],
    local_offsets [N/R+1]); see cl_moe_ep_peer_layout."""
    counts = np.ascontiguousarray(counts, np.int64)
    r, n = counts.shape
    nl = n // r
    disp = np.empty(n, np.int64)
    ret = np.empty(nl * r, np.int64)
    loc = np.empty(nl + 1, np.int64)
    rc = _lib.lib().cl_moe_ep_peer_layout(counts.ctypes.data, r, n, rank, disp.ctypes.data, ret.ctypes.data,
                                          loc.ctypes.data)
    if rc != _lib.CL_OK:
        raise MoEConfigError("ep_peer_layout: bad arguments")
    return disp, ret.reshape(nl, r), loc


def ep_group_forward(layers, hidden):
    """Single-device emulation of an R-rank expert-parallel group over the peer transport:
    layers[r] holds rank r's experts (ep_size = R, ep_rank = r); hidden[r] is rank r's batch."""
    R = len(layers)
    hidden = [lay._bf16(x) for lay, x in zip(layers, hidden)]
    outs = [torch.empty_like(x) for x in hidden]
    hs = (C.c_void_p * R)(*[lay.h.value for lay in layers])
    xs = (C.c_void_p * R)(*[x.data_ptr() for x in hidden])
    os_ = (C.c_void_p * R)(*[o.data_ptr() for o in outs])
    ts = (C.c_int64 * R)(*[x.shape[0] for x in hidden])
    _lib.check(_lib.lib().cl_moe_ep_group_forward(hs, R, xs, ts, os_, _stream(layers[0].device)), layers[0].h,
               "ep_group_forward")
    return outs


def ep_group_train_step(layers, hidden, d_out):
    """Single-device emulation of an R-rank EP training step over the peer transport:
    returns per rank (out, d_hidden, d_combine_w, dw_in, dw_out) (cl_moe_backward semantics)."""
    R = len(layers)
    hidden = [lay._bf16(x) for lay, x in zip(layers, hidden)]
    d_out = [lay._bf16(g) for lay, g in zip(layers, d_out)]
    outs = [torch.empty_like(x) for x in hidden]
    dhs = [torch.empty_like(x) for x in hidden]
    cfg = layers[0].cfg
    nl, d, f, k = cfg.n_experts // cfg.ep_size, cfg.d_model, cfg.d_ff, cfg.top_k
    dev = layers[0].device
    dcw = [torch.empty(x.shape[0], k, dtype=torch.float32, device=dev) for x in hidden]
    dwi = [torch.empty(nl, d, 2 * f, dtype=torch.float32, device=dev) for _ in range(R)]
    dwo = [torch.empty(nl, f, d, dtype=torch.float32, device=dev) for _ in range(R)]

    def arr(ts):
        return (C.c_void_p * R)(*[t.data_ptr() for t in ts])
    hs = (C.c_void_p * R)(*[lay.h.value for lay in layers])
    ts = (C.c_int64 * R)(*[x.shape[0] for x in hidden])
    _lib.check(_lib.lib().cl_moe_ep_group_train_step(hs, R, arr(hidden), ts, arr(outs), arr(d_out), arr(dhs), arr(dcw),
                                                     arr(dwi), arr(dwo), _stream(dev)), layers[0].h,
               "ep_group_train_step")
    return [(outs[r], dhs[r], dcw[r], dwi[r], dwo[r]) for r in range(R)]
