"""CPU: the balance_calibration oracle on the SPEC.md:536-544 examples, and the reference's own
checkpoint code (oracle/_ref, proj/src/checkpoint.cpp) against a plain-Python CLCKPT1 reader."""
import json
import struct

import numpy as np
import pytest

from oracle.oracle import OracleError


def read_clckpt(path):
    """CLCKPT1 (proj/include/compasslab/checkpoint.hpp:4-9) -> (header text, {name: array})."""
    blob = open(path, "rb").read()
    assert blob[:8] == b"CLCKPT1\0"
    (hl,) = struct.unpack("<Q", blob[8:16])
    header = blob[16:16 + hl].decode()
    out = {}
    for name, e in json.loads(header)["tensors"].items():
        n = int(np.prod(e["shape"])) if e["shape"] else 1
        a = np.frombuffer(blob, np.float32, n, 16 + hl + e["offset"])
        out[name] = a.reshape(e["shape"])
    return header, out


def two_expert_skew(n_base=100, frac=0.9, n_pool=400, d=8, seed=0):
    """Sign of feature 0 picks the expert: w_r[0] = (+1, -1)."""
    rng = np.random.default_rng(seed)
    wr = np.zeros((d, 2), np.float32)
    wr[0] = [1.0, -1.0]

    def toks(m, p0):
        x = rng.standard_normal((m, d)).astype(np.float32)
        s = np.where(rng.random(m) < p0, 1.0, -1.0).astype(np.float32)
        x[:, 0] = s * (0.5 + np.abs(x[:, 0]))
        return x

    base = toks(n_base, 1.0)
    base[: round(n_base * (1 - frac)), 0] *= -1  # exactly 10% to expert 1
    return base, toks(n_pool, 0.5), wr


def test_balance_already_balanced(oracle_port):
    base, pool, wr = two_expert_skew(frac=0.5)
    sel, cnt = oracle_port.balance_calibration(base, pool, wr, 1, tau=50)
    assert sel.size == 0 and cnt.tolist() == [50, 50]


def test_balance_90_10_skew(oracle_port):
    base, pool, wr = two_expert_skew()
    sel, cnt = oracle_port.balance_calibration(base, pool, wr, 1, tau=50)
    assert cnt.min() >= 50 and cnt.tolist() == [90, 50]
    assert sel.size == 40 and (pool[sel, 0] < 0).all()  # only deficit-expert tokens were taken


def test_balance_unreachable_expert(oracle_port):
    base, pool, wr = two_expert_skew()
    pool[:, 0] = np.abs(pool[:, 0])  # nothing in the pool routes to expert 1
    with pytest.raises(OracleError, match="expert 1"):
        oracle_port.balance_calibration(base, pool, wr, 1, tau=50)


def test_balance_tau_precondition(oracle_port):
    base, pool, wr = two_expert_skew()
    with pytest.raises(OracleError, match="tau"):
        oracle_port.balance_calibration(base, pool, wr, 1, tau=0)


def test_reference_checkpoint_roundtrip(oracle_ref, tmp_path):
    rng = np.random.default_rng(1)
    ts = {"layers.0.moe.router": rng.standard_normal((16, 4)).astype(np.float32),
          "layers.0.moe.experts.0.w_in": rng.standard_normal((16, 8)).astype(np.float32),
          "layers.0.moe.experts.1.w_in": rng.standard_normal((16, 8)).astype(np.float32)}
    p1, p2 = str(tmp_path / "a.ckpt"), str(tmp_path / "b.ckpt")
    oracle_ref.ckpt_write(p1, ts)
    oracle_ref.ckpt_resave(p1, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    header, got = read_clckpt(p1)
    # nlohmann dump: compact, object keys sorted -> "offset" before "shape", names in map order
    assert header.startswith('{"tensors":{"layers.0.moe.experts.0.w_in":{"offset":0,"shape":[16,8]}')
    for k, v in ts.items():
        assert np.array_equal(got[k], v)


def test_reference_checkpoint_rejects_garbage(oracle_ref, tmp_path):
    p = tmp_path / "bad.ckpt"
    p.write_bytes(b"NOTACKPT" + b"\0" * 16)
    with pytest.raises(OracleError, match="not a checkpoint"):
        oracle_ref.ckpt_resave(str(p), str(tmp_path / "out.ckpt"))
