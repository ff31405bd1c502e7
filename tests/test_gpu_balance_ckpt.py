"""GPU: balance_calibration and the reference checkpoint format (CLCKPT1,
proj/include/compasslab/checkpoint.hpp) through the C ABI.

balance_calibration selections and counts are bit-exact against the oracle (routing is bit-exact).
Checkpoints: a file written by the reference's own save_checkpoint (oracle/_ref) loads into a
layer whose forward is bit-identical to one built from the same arrays, and the layer's
save_checkpoint output is byte-identical to the reference's writer on the same tensors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle.oracle import make_inputs  # noqa: E402
from test_balance_ckpt_cpu import read_clckpt, two_expert_skew  # noqa: E402

PREFIX = "layers.3.moe."


def _cfg(d, n, k, f, t):
    from paper_2509_09121_b200.moe import MoEConfig
    return MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t)


def _layer(inp, k, t, **kw):
    from paper_2509_09121_b200.moe import MoELayer
    n, d, f2 = inp["w_in"].shape
    return MoELayer(_cfg(d, n, k, f2 // 2, t), inp["w_router"], inp["w_in"], inp["w_out"], **kw)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(torch.bfloat16)


@pytest.mark.parametrize("n,k,tau,nb,npool", [(8, 2, 40, 96, 600), (16, 4, 30, 50, 700), (32, 1, 5, 0, 900)])
def test_balance_matches_oracle(oracle_port, n, k, tau, nb, npool):
    inp = make_inputs(nb + npool, 256, n, 128, skew=1.5, experts=False)
    inp["w_in"] = np.zeros((n, 256, 256), np.float32)
    inp["w_out"] = np.zeros((n, 128, 256), np.float32)
    base, pool = inp["x"][:nb], inp["x"][nb:]
    lay = _layer(inp, k, 256)
    try:
        ref = oracle_port.balance_calibration(base if nb else None, pool, inp["w_router"], k, tau)
    except Exception as e:  # the oracle's error must be reproduced
        with pytest.raises(RuntimeError, match=str(e).split(" at ")[0]):
            lay.balance_calibration(_dev(base) if nb else None, _dev(pool), tau)
        return
    sel, cnt = lay.balance_calibration(_dev(base) if nb else None, _dev(pool), tau)
    assert np.array_equal(sel, ref[0]) and np.array_equal(cnt, ref[1])
    assert cnt.min() >= tau


def _skew_layer(d=256):
    base, pool, wr8 = two_expert_skew(d=8)
    pad = lambda x: np.pad(x, ((0, 0), (0, d - x.shape[1])))  # noqa: E731
    wr = np.zeros((d, 2), np.float32)
    wr[:8] = wr8
    inp = dict(w_router=wr, w_in=np.zeros((2, d, 256), np.float32), w_out=np.zeros((2, 128, d), np.float32))
    return _layer(inp, 1, 512), pad(base), pad(pool)


def test_balance_spec_examples(oracle_port):
    lay, base, pool = _skew_layer()
    sel, cnt = lay.balance_calibration(_dev(base), _dev(pool), 50)  # 90/10 skew, tau=50
    assert cnt.tolist() == [90, 50] and sel.size == 40 and (pool[sel, 0] < 0).all()
    sel, cnt = lay.balance_calibration(_dev(np.concatenate([base, pool[sel]])), _dev(pool), 50)  # balanced
    assert sel.size == 0 and cnt.tolist() == [90, 50]
    pool[:, 0] = np.abs(pool[:, 0])
    with pytest.raises(RuntimeError, match="expert 1"):
        lay.balance_calibration(_dev(base), _dev(pool), 50)
    from paper_2509_09121_b200._lib import MoEConfigError
    with pytest.raises(MoEConfigError, match="tau"):
        lay.balance_calibration(_dev(base), _dev(pool), 0)


def _tensors(inp, prefix=PREFIX):
    ts = {prefix + "router": inp["w_router"]}
    for e in range(inp["w_in"].shape[0]):
        ts[f"{prefix}experts.{e}.w_in"] = inp["w_in"][e]
        ts[f"{prefix}experts.{e}.w_out"] = inp["w_out"][e]
    return ts


def test_checkpoint_load_and_save_match_reference(oracle_ref, tmp_path):
    t, k = 300, 2
    inp = make_inputs(t, 256, 8, 256)  # bf16-valued weights: the layer stores them exactly
    src, mine, again = (str(tmp_path / p) for p in ("ref.ckpt", "mine.ckpt", "again.ckpt"))
    oracle_ref.ckpt_write(src, _tensors(inp))
    from paper_2509_09121_b200.moe import MoELayer
    a = _layer(inp, k, t)
    b = MoELayer(_cfg(256, 8, k, 256, t), checkpoint=src, prefix=PREFIX)
    x = _dev(inp["x"])
    assert torch.equal(a.forward(x), b.forward(x))
    b.save_checkpoint(mine, prefix=PREFIX)
    assert open(mine, "rb").read() == open(src, "rb").read()  # byte-identical to the reference writer
    oracle_ref.ckpt_resave(mine, again)
    assert open(again, "rb").read() == open(mine, "rb").read()
    _, got = read_clckpt(mine)
    for name, v in _tensors(inp).items():
        assert np.array_equal(got[name], v), name


def test_checkpoint_errors(oracle_ref, tmp_path):
    from paper_2509_09121_b200.moe import MoELayer
    inp = make_inputs(8, 256, 4, 128)
    ts = _tensors(inp, "")
    p = str(tmp_path / "x.ckpt")
    del ts["experts.3.w_out"]
    oracle_ref.ckpt_write(p, ts)
    with pytest.raises(RuntimeError, match="no tensor 'experts.3.w_out'"):
        MoELayer(_cfg(256, 4, 2, 128, 8), checkpoint=p)
    ts = _tensors(inp, "")
    ts["router"] = ts["router"][:, :2]
    oracle_ref.ckpt_write(p, ts)
    with pytest.raises(RuntimeError, match="unexpected shape"):
        MoELayer(_cfg(256, 4, 2, 128, 8), checkpoint=p)
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"garbage" * 4)
    with pytest.raises(RuntimeError, match="not a checkpoint"):
        MoELayer(_cfg(256, 4, 2, 128, 8), checkpoint=str(bad))


def test_checkpoint_expert_shard(oracle_ref, tmp_path):
    """An EP rank loads only its contiguous expert shard and saves it under global expert ids."""
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer
    inp = make_inputs(8, 256, 8, 128)
    p, q = str(tmp_path / "all.ckpt"), str(tmp_path / "r1.ckpt")
    oracle_ref.ckpt_write(p, _tensors(inp))
    cfg = MoEConfig(d_model=256, n_experts=8, top_k=2, d_ff=128, max_tokens=8, ep_size=2, ep_rank=1)
    MoELayer(cfg, checkpoint=p, prefix=PREFIX).save_checkpoint(q, prefix=PREFIX)
    _, got = read_clckpt(q)
    assert sorted(got) == sorted([PREFIX + "router"] + [f"{PREFIX}experts.{e}.{w}" for e in range(4, 8)
                                                        for w in ("w_in", "w_out")])
    for e in range(4, 8):
        assert np.array_equal(got[f"{PREFIX}experts.{e}.w_in"], inp["w_in"][e])


def test_collect_calibration_counts(oracle_port):
    """SPEC.md:532-536 collect_calibration: counts sum = B*K, equal to the oracle's routing counts
    accumulated over batches (skewed router included); an empty token set gives zero counts."""
    n, k, d = 16, 4, 256
    inp = make_inputs(900, d, n, 256, skew=1.8)
    lay = _layer(inp, k, 512)
    x = inp["x"]
    lay.calibrate(_dev(x[:0]), reset=True)
    st = lay.calibration_stats()
    assert st["counts"].sum() == 0 and st["x_max"].max() == 0
    lay.calibrate(_dev(x[:500]), reset=True)
    lay.calibrate(_dev(x[500:]), reset=False)
    st = lay.calibration_stats()
    ref = oracle_port.route(x, inp["w_router"], k)["counts"]
    assert st["counts"].sum() == 900 * k
    assert np.array_equal(st["counts"], ref)
    assert np.array_equal(st["ch_max"], np.abs(x).max(0))
    assert ref[0] / ref.sum() > 2.0 / n  # the injected skew is visible in the statistics
