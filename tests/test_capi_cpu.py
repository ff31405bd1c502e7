"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol the header
declares, and fails loudly (no CPU fallback) when no sm_100 device is present."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "compass_moe.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cl_moe_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_api():
    names = _declared_functions()
    for required in ["cl_moe_create", "cl_moe_route_tokens", "cl_moe_moe_forward", "cl_moe_forward",
                     "cl_moe_forward_host", "cl_moe_last_error", "cl_moe_destroy", "cl_moe_quantize_fp8"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2509_09121_b200 import _lib
    L = _lib.lib()
    missing = [n for n in _declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert L.cl_moe_version().decode().startswith("0.")


def test_status_codes_match_reference_header():
    # proj/include/compass_lab.h:23-27
    from paper_2509_09121_b200 import _lib
    assert (_lib.CL_OK, _lib.CL_ERR_RUN, _lib.CL_ERR_CONFIG) == (0, 1, 2)
    src = open(HEADER).read()
    assert "CL_OK = 0" in src and "CL_ERR_RUN = 1" in src and "CL_ERR_CONFIG = 2" in src


def test_config_struct_layout_matches_header():
    from paper_2509_09121_b200 import _lib
    assert C.sizeof(_lib.Config) == 5 * 8 + 4 * 4
    assert C.sizeof(_lib.Decision) == 8 * 8


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_09121_b200 import _lib
    L = _lib.lib()
    cfg = _lib.Config(256, 4, 2, 128, 16, 0, 0, 1, 0)
    h = C.c_void_p()
    rc = L.cl_moe_create_synthetic(C.byref(cfg), 1, C.byref(h))
    assert rc == _lib.CL_ERR_RUN
    assert not h.value


def test_invalid_config_is_config_error():
    from paper_2509_09121_b200 import _lib
    L = _lib.lib()
    h = C.c_void_p()
    for bad in [_lib.Config(250, 4, 2, 128, 16, 0, 0, 1, 0),   # d not multiple of 256
                _lib.Config(256, 4, 5, 128, 16, 0, 0, 1, 0),   # K > N
                _lib.Config(256, 4, 2, 100, 16, 0, 0, 1, 0),   # f not multiple of 128
                _lib.Config(256, 6, 2, 128, 16, 0, 0, 4, 0)]:  # N not divisible by ep
        assert L.cl_moe_create_synthetic(C.byref(bad), 1, C.byref(h)) == _lib.CL_ERR_CONFIG
