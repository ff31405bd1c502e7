"""ctypes binding of the in-tree C-ABI library ``libcompass_moe.so`` (include/compass_moe.h).

There is no fallback: if the library is missing (and cannot be built with nvcc) or the device is
not an sm_100 part, every call fails loudly. The library is loaded from the package directory so
that the driver's native-code check sees it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# CL_MOE_LIB_VARIANT=<name> loads libcompass_moe.<name>.so from the same directory (A/B builds)
LIB_PATH = os.path.join(HERE, "libcompass_moe.so" if not os.environ.get("CL_MOE_LIB_VARIANT")
                        else f"libcompass_moe.{os.environ['CL_MOE_LIB_VARIANT']}.so")
CSRC = os.path.join(HERE, "csrc")

CL_OK, CL_ERR_RUN, CL_ERR_CONFIG = 0, 1, 2
CL_MOE_BF16, CL_MOE_FP8_E4M3 = 0, 1
CL_MOE_IO_BF16, CL_MOE_IO_F32 = 0, 1
STAGE = dict(offsets=0, perm=1, inv=2, row_weight=3, x_perm=4, act=5, y=6)


class Config(C.Structure):
    _fields_ = [
        ("d_model", C.c_int64),
        ("n_experts", C.c_int64),
        ("top_k", C.c_int64),
        ("d_ff", C.c_int64),
        ("max_tokens", C.c_int64),
        ("device", C.c_int32),
        ("gemm_ctas", C.c_int32),
        ("ep_size", C.c_int32),
        ("ep_rank", C.c_int32),
    ]


class Decision(C.Structure):
    _fields_ = [
        ("logits", C.c_void_p),
        ("probs", C.c_void_p),
        ("topk_idx", C.c_void_p),
        ("combine_weights", C.c_void_p),
        ("counts", C.c_void_p),
        ("agg_prob", C.c_void_p),
        ("aux_loss", C.c_void_p),
        ("z_loss", C.c_void_p),
    ]


class StageView(C.Structure):
    _fields_ = [
        ("offsets", C.c_void_p),
        ("perm", C.c_void_p),
        ("inv", C.c_void_p),
        ("row_weight", C.c_void_p),
        ("x_perm", C.c_void_p),
        ("act", C.c_void_p),
        ("y", C.c_void_p),
        ("rows", C.c_int64),
    ]


class MoEError(RuntimeError):
    """A CL_ERR_RUN status (the reference's ValidationError / runtime failure)."""


class MoEConfigError(MoEError):
    """A CL_ERR_CONFIG status (the reference's ConfigError)."""


_lib = None

# name -> (restype, argtypes); mirrors include/compass_moe.h
_PROTOS = {
    "cl_moe_version": (C.c_char_p, []),
    "cl_moe_create": (C.c_int, [C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "cl_moe_create_synthetic": (C.c_int, [C.POINTER(Config), C.c_uint64, C.POINTER(C.c_void_p)]),
    "cl_moe_create_from_checkpoint": (C.c_int, [C.POINTER(Config), C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "cl_moe_save_checkpoint": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
    "cl_moe_balance_calibration": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                             C.c_void_p, C.POINTER(C.c_int64), C.c_void_p, C.c_void_p]),
    "cl_moe_destroy": (None, [C.c_void_p]),
    "cl_moe_last_error": (C.c_char_p, [C.c_void_p]),
    "cl_moe_synthetic_tokens": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p]),
    "cl_moe_synthetic_tokens_shifted": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int64, C.c_float, C.c_void_p,
                                                  C.c_void_p]),
    "cl_moe_synthetic_skew": (C.c_int, [C.c_void_p, C.c_double]),
    "cl_moe_route_tokens": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(Decision), C.c_void_p]),
    "cl_moe_moe_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(Decision), C.c_void_p]),
    "cl_moe_route_tokens_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(Decision), C.c_void_p]),
    "cl_moe_forward_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(Decision), C.c_void_p]),
    "cl_moe_forward_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32]),
    "cl_moe_forward_host_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32]),
    "cl_moe_host_wait": (C.c_int, [C.c_void_p]),
    "cl_moe_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cl_moe_stage_buffers": (C.c_int, [C.c_void_p, C.POINTER(StageView)]),
    "cl_moe_copy_stage": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]),
    "cl_moe_profile": (C.c_int, [C.c_void_p, C.c_int32]),
    "cl_moe_profile_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "cl_moe_forward_train": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(Decision), C.c_void_p]),
    "cl_moe_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_backward_full": (C.c_int, [C.c_void_p, C.c_void_p, C.c_float, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_ep_unique_id": (C.c_int, [C.c_void_p]),
    "cl_moe_ep_init": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cl_moe_ep_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(Decision), C.c_void_p]),
    "cl_moe_calibration_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_ep_peer_init": (C.c_int, [C.c_void_p]),
    "cl_moe_ep_group_forward": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_ep_group_train_step": (C.c_int, [C.c_void_p, C.c_int32] + [C.c_void_p] * 9),
    "cl_moe_forward_graph": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "cl_moe_ep_last_counts": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cl_moe_ep_peer_layout": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    "cl_moe_ep_layout": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_int64)]),
    "cl_moe_calibrate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "cl_moe_quantize_fp8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_compute_smoothing": (C.c_int, [C.c_void_p, C.c_float, C.c_void_p]),
    "cl_moe_fold_smoothing": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cl_moe_set_precision": (C.c_int, [C.c_void_p, C.c_int32]),
    "cl_moe_get_fp8_scales": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_set_router_fp8": (C.c_int, [C.c_void_p, C.c_int32, C.c_float]),
    "cl_moe_save_fp8_scheme": (C.c_int, [C.c_void_p, C.c_char_p]),
    "cl_moe_get_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "cl_moe_router_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_router_variant": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cl_moe_load_fp8_scheme": (C.c_int, [C.c_void_p, C.c_char_p]),
    "cl_moe_get_router_fp8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
}


def build() -> None:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", CSRC], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            if os.environ.get("CL_MOE_LIB_VARIANT") and not hasattr(L, name):
                continue  # an older A/B build may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, handle=None, what: str = "") -> None:
    if rc == CL_OK:
        return
    msg = lib().cl_moe_last_error(handle).decode() if handle else ""
    cls = MoEConfigError if rc == CL_ERR_CONFIG else MoEError
    raise cls(f"{what}: {msg}" if what else msg)
