"""Generates tests/golden/*.npz from the REFERENCE implementation (oracle/_ref: the reference's
own proj/src/tensor.cpp + common.cpp compiled from /root/reference and composed per SPEC.md by
oracle/ref_compose.cpp). Run in the build container, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The inputs are regenerated from the reference Prng streams (oracle.make_inputs, root seed
20261018), so a fixture stores only the case shape and the reference outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, make_inputs  # noqa: E402

CASES = [
    # name, T, d, N, K, f, skew
    ("small_n8_k2", 64, 64, 8, 2, 32, None),
    ("small_n16_k4", 50, 96, 16, 4, 48, None),
    ("skew_n8_k2", 80, 64, 8, 2, 32, 2.0),
    ("k1_n4", 33, 32, 4, 1, 16, None),
]


def main():
    ref = Oracle("reference")
    for name, t, d, n, k, f, skew in CASES:
        inp = make_inputs(t, d, n, f, skew=skew)
        r = ref.route(inp["x"], inp["w_router"], k)
        out = ref.moe_forward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"], r["combine_weights"], jobs=1)
        aux = ref.aux_loss(r["probs"], r["counts"], k)
        z = ref.z_loss(r["logits"])
        rows = np.where((r["topk_idx"] == 0).any(1))[0]
        dy = make_inputs(len(rows), d, 1, f, seed=7, experts=False)["x"]
        dx, dwi, dwo = ref.expert_ffn_backward(inp["x"][rows], inp["w_in"][0], inp["w_out"][0], dy)
        gl = make_inputs(t, d, 1, f, seed=11, experts=False)["x"]
        ldh, ldcw, ldwi, ldwo = ref.moe_backward(inp["x"], inp["w_in"], inp["w_out"], r["topk_idx"],
                                                 r["combine_weights"], gl)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), shape=np.array([t, d, n, k, f]),
                            layer_d_hidden=ldh, layer_d_combine_w=ldcw, layer_dw_in=ldwi, layer_dw_out=ldwo,
                            skew=np.array([np.nan if skew is None else skew]), logits=r["logits"], probs=r["probs"],
                            topk_idx=r["topk_idx"], combine_weights=r["combine_weights"], counts=r["counts"],
                            agg_prob=r["agg_prob"], aux=np.float32(aux), z=np.float32(z), out=out, bwd_rows=rows,
                            dx=dx, dw_in=dwi, dw_out=dwo)
        print("wrote", name)


if __name__ == "__main__":
    main()
