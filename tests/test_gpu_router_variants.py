"""Every K1 router variant (ws and lat 1x1 chains, small 1x4 with a deep prefetch ring, big 2x4 / 4x4, dmma on the
fp64 tensor cores), forced through
CL_MOE_ROUTER in a fresh process, gives bit-exact logits / top-k / counts against the oracle,
including ragged last tiles, shapes where the automatic choice would pick another variant, and exact
ties (duplicated router columns, all-zero tokens: the lowest expert index must win). Each case runs
three times: bf16 tokens; unrounded fp32 tokens through the fp32 router input; and the router of the
FP8 scheme (E4M3 codes of x / s_x widened in K1, qdq'd W_r) against router_fp8_sim. The "lat"
variant is bf16-only; forced with another input it runs ws. "dmma" (N <= 32) falls back to the automatic choice for
more experts."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("variant", ["small", "big2", "big4", "lat", "ws", "dmma"])
@pytest.mark.parametrize("t,d,n,k,mode", [(333, 256, 16, 2, "random"), (1000, 512, 8, 2, "random"),
                                          (257, 256, 32, 4, "random"), (70, 1024, 4, 1, "random"),
                                          (5, 256, 128, 8, "random"), (300, 256, 16, 4, "ties"),
                                          (90, 256, 128, 8, "ties"), (2400, 256, 4, 2, "random")])
@pytest.mark.parametrize("dtype", ["bf16", "f32", "fp8"])
def test_router_variant_bit_exact(variant, t, d, n, k, mode, dtype):
    env = dict(os.environ, CL_MOE_ROUTER=variant.rstrip("24"), PYTHONPATH=ROOT)
    if variant.startswith("big"):
        env["CL_MOE_BIG_TOK"] = variant[-1]  # 2 or 4 tokens x 4 experts per thread
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "route_check.py"), str(t), str(d), str(n),
                        str(k), mode, dtype], env=env, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
