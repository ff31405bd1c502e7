"""Grouped GEMMs on clusters of two CTA pairs that share the B (weight) tile through TMA multicast
(CL_MOE_GEMM_MC=1, grouped_gemm_kernel<..., kCM = 2>). Each output tile is still one pair's
tcgen05 MMAs over the same K order, so GEMM1 (+SwiGLU) and GEMM2 outputs must be bit-identical to
the single-pair kernels — bf16 and FP8, with experts whose m-tile count is odd (the cluster's
second pair idles on that tile but still streams its share of B), tail tiles of <= 128 rows (half
tiles) and a skewed expert. Fresh processes (the switch is read once); a hang is bounded by a
timeout."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, mc, shape):
    env = dict(os.environ, PYTHONPATH=ROOT, CL_MOE_GEMM_MC="1" if mc else "0")
    path = str(tmp_path / f"mc_{mc}.npz")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "mc_run.py"), path, *map(str, shape)],
                       env=env, capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    return np.load(path)


@pytest.mark.parametrize("shape", [(6000, 512, 8, 2, 512), (5000, 256, 4, 2, 1024), (9000, 512, 16, 2, 256),
                                   (2500, 1024, 2, 1, 768)])
def test_multicast_clusters_bit_identical(tmp_path, shape):
    a = _run(tmp_path, True, shape)
    b = _run(tmp_path, False, shape)
    for name in b.files:
        assert np.array_equal(a[name], b[name]), name
