"""Subprocess helper for tests/test_gpu_ep.py::test_ep_stalled_exchange_times_out: with
CL_MOE_EP_TEST_STALL_MS (a kernel that spins at the end of every expert-parallel forward, standing
in for a stalled peer) longer than CL_MOE_EP_TIMEOUT_S, cl_moe_sync returns CL_ERR_RUN instead of
hanging, the communicator is aborted, later EP calls fail with the same reason, and cl_moe_ep_init
restores a working communicator."""
import sys
import time

import numpy as np
import torch

from oracle.oracle import make_inputs
from paper_2509_09121_b200.moe import MoEConfig, MoEError, MoELayer


def main(transport):
    t, d, n, k, f = 300, 256, 4, 2, 256
    inp = make_inputs(t, d, n, f)
    lay = MoELayer(MoEConfig(d_model=d, n_experts=n, top_k=k, d_ff=f, max_tokens=t), inp["w_router"], inp["w_in"],
                   inp["w_out"])
    lay.ep_init(MoELayer.ep_unique_id())
    if transport == "peer":
        lay.ep_peer_init()
    x = torch.from_numpy(inp["x"]).cuda().to(torch.bfloat16).contiguous()
    lay.ep_forward(x)
    t0 = time.time()
    try:
        lay.sync()
        print("NO TIMEOUT")
        return 1
    except MoEError as e:
        msg = str(e)
    waited = time.time() - t0
    # detected after the 1 s limit; the call returns once ncclCommAbort is done (it drains the
    # device work queued behind the stalled kernel), well before any hang would be noticed
    if "timed out after 1 s" not in msg or "aborted" not in msg or waited > 15.0:
        print("BAD", msg, waited)
        return 1
    try:
        lay.ep_forward(x)
        print("EP CALL AFTER ABORT DID NOT FAIL")
        return 1
    except MoEError as e:
        if "timed out" not in str(e):
            print("BAD REASON", e)
            return 1
    torch.cuda.synchronize()  # the stalled kernel finishes; the device is healthy
    lay.ep_init(MoELayer.ep_unique_id())
    out = lay.ep_forward(x)
    torch.cuda.synchronize()
    lay.sync()
    ref = lay.forward(x)  # 1-rank: the EP path is the loopback of the single-GPU layer
    torch.cuda.synchronize()
    lay.sync()
    dl = (out.float() - ref.float()).abs().max().item()
    if not np.isfinite(dl) or dl > 2e-2 * ref.float().abs().max().item():
        print("BAD OUTPUT", dl)
        return 1
    print("ok", f"{waited:.2f}s")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
