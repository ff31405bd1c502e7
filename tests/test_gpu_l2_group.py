"""The L2-resident tile order of the grouped GEMMs (host_forward.cuh m_group_for / launch_gemm;
grouped_gemm.cuh tile decode): an expert's m-tiles run in groups of `m_group` (budget
CL_MOE_L2_GROUP_MB of A rows, floored at CL_MOE_GEMM_GROUP_MIN / CL_MOE_WGRAD_GROUP_MIN, default 4 / 6),
each group sweeping every n-block. At the default 32 MB budget and small test shapes every expert
fits one group, so the grouped order is only reached at the benchmarked shapes (C2 GEMM2, C3, the
hot C5 expert) — here it is forced with CL_MOE_L2_GROUP_MB=1 in a fresh process, once with the
default floors (groups of 4 or 6 m-tiles, uneven last groups) and once with the floor at 1 (m_group = 2 at
d = 1024 and 1 for K = 2816 rows). The tile order changes nothing a tile computes (every output
element keeps its K order), so bf16 forward, FP8 forward and the training step (dgrad GEMMs and the
weight-gradient GEMMs' groups) must be bit-identical to the default order, and the forward within
tolerance of the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, mb, shape, floor=None):
    env = dict(os.environ, PYTHONPATH=ROOT)
    if mb is not None:
        env["CL_MOE_L2_GROUP_MB"] = str(mb)
    if floor is not None:
        env["CL_MOE_GEMM_GROUP_MIN"] = env["CL_MOE_WGRAD_GROUP_MIN"] = str(floor)
    path = str(tmp_path / f"run_{mb}_{floor}.npz")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "l2group_run.py"), path,
                        *map(str, shape)], env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    return np.load(path)


@pytest.mark.parametrize("shape", [(8192, 1024, 4, 2, 2816), (6000, 512, 8, 2, 1024)])
def test_forced_l2_groups_bit_identical(tmp_path, shape):
    from oracle.oracle import Oracle, make_inputs
    grouped = _run(tmp_path, 1, shape)
    small = _run(tmp_path, 1, shape, floor=1)
    plain = _run(tmp_path, None, shape)
    for name in plain.files:
        assert np.array_equal(grouped[name], plain[name]), name
        assert np.array_equal(small[name], plain[name]), name
    t, d, n, k, f = shape
    inp = make_inputs(t, d, n, f)
    o = Oracle("port")
    r = o.route(inp["x"], inp["w_router"], k)
    ref = o.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"],
                        jobs=os.cpu_count() or 1)
    out = (grouped["out_bf16"].astype(np.int32) << 16).view(np.float32).astype(np.float64)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-2
