"""The compiled reference-side consumer (tests/integration/consumer.cpp, the INTEGRATION.md C++
snippet) linked against libcompass_moe.so, run on the GPU: the drop-in host call on fp32 buffers,
the status-code mapping of proj/src/capi.cpp:57-63 (ConfigError -> CL_ERR_CONFIG, everything else
-> CL_ERR_RUN, last_error "" after a success), and its output equal to the Python binding's and
within tolerance of the oracle (routing on the fp32 values, bit-exact)."""
import os
import shutil
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


def test_cpp_consumer_runs_drop_in_call(tmp_path):
    from oracle.oracle import Oracle, make_inputs
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    if not shutil.which("g++"):
        pytest.skip("g++ absent")
    lib = os.path.join(ROOT, "paper_2509_09121_b200", "libcompass_moe.so")
    extra = [f"-I{REF_INC}", "-DCOMPASS_HAVE_LAB"] if os.path.exists(os.path.join(REF_INC, "compass_lab.h")) else []
    exe = str(tmp_path / "consumer")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", f"-I{os.path.join(ROOT, 'include')}", *extra,
                        os.path.join(ROOT, "tests", "integration", "consumer.cpp"), lib,
                        f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    t, d, n, k, f = 300, 512, 8, 2, 256
    inp = make_inputs(t, d, n, f, bf16=False)  # unrounded fp32 tokens, as the reference's Tensors
    src = str(tmp_path / "in.bin")
    with open(src, "wb") as fh:
        np.array([d, n, k, f, t], np.int64).tofile(fh)
        for a in (inp["w_router"], inp["w_in"], inp["w_out"], inp["x"]):
            np.ascontiguousarray(a, np.float32).tofile(fh)
    dst = str(tmp_path / "out.bin")
    r = subprocess.run([exe, src, dst], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
    out = np.fromfile(dst, np.float32).reshape(t, d)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), inp["w_router"], inp["w_in"],
                   inp["w_out"])
    assert np.array_equal(out, lay.forward_host(inp["x"], "f32"))
    lay.close()
    o = Oracle("port")
    rr = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], rr["topk_idx"], rr["combine_weights"])
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-2
