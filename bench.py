#!/usr/bin/env python3
"""Benchmark of the MoE-layer hot path (BASELINE.json metric) on B200.

Default workload = BASELINE.json configs[1] ("C2"): one bf16 MoE layer, T=16384 tokens, d=4096,
N=16 experts, top-2, SwiGLU FFN 14336, synthetic tokens and random-init weights drawn on the
device with the reference counter PRNG (root seed 20261018).

A step = one full layer forward (router -> plan -> dispatch -> GEMM1+SwiGLU -> GEMM2+weight ->
combine) over one batch of T tokens, inputs resident in HBM (x = 134 MB and 5.6 GB of weights:
every input is larger than the 126 MB L2, so no flush is needed between steps).

Prints ONE JSON line (rank 0). ``--impl reference`` times the reference CPU implementation
(oracle/_ref: the reference's own tensor.cpp compiled from /root/reference, composed per SPEC)
on a bounded token sample of the same layer on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]
    "c2": dict(workload="single-B200 MoE layer bf16 (BASELINE configs[1])", T=16384, d=4096, N=16, K=2, f=14336),
    # BASELINE.json configs[0] shape on the GPU
    "c1": dict(workload="small MoE layer (BASELINE configs[0] shape) bf16 on GPU", T=4096, d=1024, N=8, K=2, f=2816),
    # BASELINE.json configs[2]: Compass-v3-shaped layer (N=16, K=4; d, f derived in SURVEY §8d),
    # 8192 tokens per rank (65536 over 8 EP ranks)
    "c3": dict(workload="Compass-v3-shaped MoE layer, EP over the ranks (BASELINE configs[2])", T=8192, d=8192, N=16,
               K=4, f=12288),
    # BASELINE.json configs[3] decode-size batch at the C2 layer shape (bf16 path)
    "c4": dict(workload="decode-size batch at the C2 layer shape (BASELINE configs[3])", T=256, d=4096, N=16, K=2,
               f=14336),
    # BASELINE.json configs[4]: skewed routing, forward + expert-FFN backward
    "c5": dict(workload="skewed-routing stress, fwd + expert-FFN bwd (BASELINE configs[4])", T=65536, d=4096, N=16,
               K=2, f=14336, skew=1.8, train=True),
}
SEED = 20261018
METRIC = "MoE-layer tokens/sec at 1/2/4/8 B200; % tcgen05 peak (GEMM), % HBM BW (dispatch)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


def fp8_peak():
    p = os.path.join(ROOT, "profiles", "fp8_peak.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)["fp8_tflops"], "measured (tools/fp8_peak.py, cuBLASLt e4m3 8192^3)"
    return 4500.0, "nominal dense"



class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50", "-i", self.gpu_id],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"], samples=0)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return dict(sm_mhz=float(np.median(sm)) if sm else None, sm_max_mhz=max(mx) if mx else None,
                    power_w_max=max(pw) if pw else None, reasons=sorted(reasons), samples=len(sm))


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n: int) -> int:
    """`bench.py --gpus N` started without a launcher: re-exec this command as N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1, the way the driver launches it."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, cwd=ROOT).returncode


def run_dry(args):
    """--dry-run: the rank plumbing only (no GPU): every rank joins a gloo group and rank 0 prints
    the world size the group actually formed (tests/test_bench_contract_cpu.py)."""
    import torch
    import torch.distributed as dist
    rank, _, world = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        formed = int(t.item())
        dist.destroy_process_group()
    else:
        formed = 1
    if rank == 0:
        print(json.dumps(dict(dry_run=True, gpus=args.gpus, world_size=world, ranks_joined=formed)), flush=True)


# ------------------------------------------------------------------------------------------
# CPU baseline: the reference implementation (or the oracle port) on a bounded token sample
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(cfg, t_sample: int, kind_pref: str = "reference"):
    """Prepare a bounded sample of the configured layer for the CPU oracle. Weights are random
    uniform values (the reference arithmetic is data-independent: dense fp64-accumulated loops),
    tokens and router weights are the §8(d) PRNG streams so routing is realistic."""
    from oracle.oracle import Oracle, available, make_inputs
    kind = "reference" if (kind_pref == "reference" and available("reference")) else "port"
    o = Oracle(kind)
    d, n, k, f = cfg["d"], cfg["N"], cfg["K"], cfg["f"]
    inp = make_inputs(t_sample, d, n, f, experts=False)
    rng = np.random.default_rng(0)
    a = np.float32(1.0 / np.sqrt(d))
    w_in = (rng.random((n, d, 2 * f), dtype=np.float32) - np.float32(0.5)) * a
    w_out = (rng.random((n, f, d), dtype=np.float32) - np.float32(0.5)) * a
    return o, kind, inp, w_in, w_out


def cpu_step(o, inp, w_in, w_out, k, jobs):
    r = o.route(inp["x"], inp["w_router"], k)
    return o.moe_forward(inp["x"], w_in, w_out, r["topk_idx"], r["combine_weights"], jobs=jobs)


def pick_cpu_tokens(cfg):
    # ~45 GFLOP per 64 tokens at the C2 shape; aim for ~5-20 s of CPU work per sample. A config
    # whose whole batch is <= 160 GFLOP (C1: 4096 tokens, 142 GFLOP, ~8-10 s on the box's host
    # threads) runs in full, as SURVEY.md §8(d) asks for the reference's own CPU shape.
    flop_per_tok = 2 * cfg["K"] * 3 * cfg["d"] * cfg["f"]
    if cfg["T"] * flop_per_tok <= 160e9:
        return int(cfg["T"])
    return int(max(8, min(cfg["T"], round(60e9 / flop_per_tok / 8) * 8)))


def run_reference(args, cfg):
    rank, _, world = dist_env()
    if rank != 0:
        return
    t_s = pick_cpu_tokens(cfg)
    jobs = os.cpu_count() or 1
    o, kind, inp, w_in, w_out = cpu_sample(cfg, t_s)
    cores = min(jobs, cfg["N"])
    for _ in range(args.warmup):
        cpu_step(o, inp, w_in, w_out, cfg["K"], jobs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_step(o, inp, w_in, w_out, cfg["K"], jobs)
    dt = time.perf_counter() - t0
    val = t_s * args.steps / dt
    sample = (f"{t_s} of {cfg['T']} tokens per step at the layer shape d={cfg['d']} N={cfg['N']} K={cfg['K']} "
              f"f={cfg['f']} (fp32, expert fan-out over {cores} threads via the reference parallel_for)")
    line = dict(metric=METRIC, value=val, unit="tokens/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
                ms_per_step=dt / args.steps * 1e3, higher_is_better=True, scaling="weak", vs_baseline=None,
                dtype="f32", data="synthetic", impl="reference",
                config=dict(workload=cfg["workload"], T=cfg["T"], d=cfg["d"], n_experts=cfg["N"], top_k=cfg["K"],
                            d_ff=cfg["f"], parallelism="cpu", sample_tokens=t_s),
                cpu_baseline=dict(value=val, unit="tokens/s", cores=cores, kind=kind, sample=sample,
                                  cpu_model=cpu_model(), host_threads=jobs),
                e2e=dict(value=val, unit="tokens/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def count_our_launches(step, sync):
    """Kernels of this library launched by one step, counted by the CUDA profiler (CUPTI, through
    torch.profiler) on one extra untimed step: kernels in the `cmoe` namespace. None when the
    profiler is unavailable."""
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            sync()
        n = sum(ev.count for ev in prof.key_averages() if "cmoe::" in ev.key)
        return n if n > 0 else None
    except Exception:  # noqa: BLE001 — the count is diagnostic; the timed run does not depend on it
        return None


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2509_09121_b200.moe import MoEConfig, MoELayer

    T, d, N, K, f = cfg["T"], cfg["d"], cfg["N"], cfg["K"], cfg["f"]
    if args.tokens:
        T = args.tokens
    elif cfg.get("train") and world > 1:
        T = cfg["T"] // world  # C5 is quoted on 65536 tokens in total, split over the EP ranks
    if world > 1 and N % world:
        raise SystemExit(f"n_experts={N} is not divisible by {world} ranks")
    layer = MoELayer(MoEConfig(d_model=d, n_experts=N, top_k=K, d_ff=f, max_tokens=T, device=local_rank,
                               gemm_ctas=args.gemm_ctas, ep_size=world, ep_rank=rank), seed=SEED)
    if world > 1:
        # expert parallelism: NCCL id from rank 0, communicator owned by the library
        obj = [MoELayer.ep_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        layer.ep_init(obj[0])
    train = bool(cfg.get("train"))
    transport = "NCCL send/recv"
    if world > 1 and args.ep_transport == "peer":
        try:
            layer.ep_peer_init()
            transport = ("NVLink peer stores: dispatch kernel + GEMM2 epilogue" +
                         (", combine-backward kernel + dgrad-2 epilogue" if train else "") + "; NCCL for counts/barriers")
        except Exception as e:  # no P2P between the devices: keep the NCCL transport, say so
            transport = f"NCCL send/recv (peer transport unavailable: {e})"
    if cfg.get("skew"):
        layer.synthetic_skew(cfg["skew"])
    x = layer.synthetic_tokens(T, SEED + rank, shift=1.0 if cfg.get("skew") else 0.0)
    out = torch.empty_like(x)
    if train:
        g_out = layer.synthetic_tokens(T, SEED + 7 + rank)
        d_hid = torch.empty_like(x)
        nl_ = N // world
        d_cw = torch.empty(T, K, dtype=torch.float32, device=x.device)
        dwi = torch.empty(nl_, d, 2 * f, dtype=torch.float32, device=x.device)
        dwo = torch.empty(nl_, f, d, dtype=torch.float32, device=x.device)
    if args.precision == "fp8":
        # expert-aware FP8: calibrate on this batch (per-expert activation maxima), quantize weights
        layer.calibrate(x)
        layer.quantize_fp8()
    stream = torch.cuda.current_stream()

    def step(xb=None, gb=None, ob=None, dhb=None):
        if train:
            xb = x if xb is None else xb
            gb = g_out if gb is None else gb
            ob = out if ob is None else ob
            dhb = d_hid if dhb is None else dhb
            layer._check(layer.L.cl_moe_forward_train(layer.h, xb.data_ptr(), T, ob.data_ptr(), None,
                                                      stream.cuda_stream), "forward_train")
            layer._check(layer.L.cl_moe_backward(layer.h, gb.data_ptr(), dhb.data_ptr(), d_cw.data_ptr(),
                                                 dwi.data_ptr(), dwo.data_ptr(), stream.cuda_stream), "backward")
        else:
            layer._check(layer.L.cl_moe_forward(layer.h, x.data_ptr(), T, out.data_ptr(), None, stream.cuda_stream),
                         "forward")

    for _ in range(args.warmup):
        step()
    layer.sync()

    props = torch.cuda.get_device_properties(local_rank)
    sampler = ClockSampler("GPU-" + str(props.uuid) if getattr(props, "uuid", None) else str(local_rank))
    layer.profile(True)
    sampler.start()
    time.sleep(0.3)  # let the sampler attach
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    layer.sync()
    ms = ev0.elapsed_time(ev1)
    stage_ms, calls = layer.profile_read()
    layer.profile(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    value = world * T * args.steps / (ms / 1e3)

    if train:
        # double-buffered pipeline: H2D of step i+1 and D2H of step i-1 on copy streams overlap
        # step i's compute; every step still moves its inputs in and its outputs out
        xh = torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True)
        gh = torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True)
        oh = [torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
        dh_h = [torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
        xh.copy_(x)
        gh.copy_(g_out)
        xs_, gs_ = [x, torch.empty_like(x)], [g_out, torch.empty_like(x)]
        os_, dhs_ = [out, torch.empty_like(x)], [d_hid, torch.empty_like(x)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_drained = [torch.cuda.Event() for _ in range(2)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_steps = max(2, args.steps // 2)
        for i in range(e2e_steps):
            b = i % 2
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(ev_done[b])  # step i-2 no longer reads this input set
                xs_[b].copy_(xh, non_blocking=True)
                gs_[b].copy_(gh, non_blocking=True)
                ev_in[b].record(s_in)
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_drained[b])  # step i-2's outputs are out of this set
            step(xs_[b], gs_[b], os_[b], dhs_[b])
            ev_done[b].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[b])
                oh[b].copy_(os_[b], non_blocking=True)
                dh_h[b].copy_(dhs_[b], non_blocking=True)
                ev_drained[b].record(s_out)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e_val = world * T * e2e_steps / e2e_s
        h2d_b, d2h_b = 2 * T * d * 2, 2 * T * d * 2
    else:
        h2d_b, d2h_b = T * d * 2, T * d * 2
    # ---- end to end through the host-buffer C-ABI (pinned host bf16 in/out, pipelined calls) ----
    xh = [torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)] if not train else []
    for b in xh:
        b.copy_(x)
    if not train:
        oh = [torch.empty(T, d, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
        for i in range(2):
            layer.forward_host_async(xh[i].data_ptr(), T, oh[i].data_ptr())
        layer.host_wait()
        # at least 50 calls so the 2-slot pipeline's fill (first H2D) and drain (last D2H) are
        # amortised the way a serving loop amortises them; every call still copies in and out
        e2e_steps = max(args.steps, 50)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            layer.forward_host_async(xh[i % 2].data_ptr(), T, oh[i % 2].data_ptr())
        layer.host_wait()
        e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = world * T * e2e_steps / e2e_s

    # ---- our kernel launches per step, counted (CUPTI) on one extra untimed step ----
    per_step_launches = count_our_launches(step, layer.sync)

    # ---- NVLink exchange accounting (N > 1): exact rows this rank sent to other ranks ----
    a2a = None
    if world > 1:
        counts = layer.ep_last_counts()  # [R][N], row = source
        nl_ = N // world
        mine = counts[rank]
        remote_rows = int(sum(mine[g] for g in range(N) if g // nl_ != rank))
        esz_x = 1 if args.precision == "fp8" else 2
        b_out = remote_rows * d * esz_x                # dispatch direction (x rows)
        b_back = remote_rows * d * 2                   # return direction (bf16 rows)
        t = torch.tensor([b_out, b_back], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        a2a = dict(transport=transport, max_rank_bytes_dispatch=float(t[0]), max_rank_bytes_return=float(t[1]),
                   dispatch_stage_gbs_rank0=float(t[0]) / max(stage_ms["dispatch"] / max(calls[0], 1), 1e-9) / 1e6,
                   note="bytes of the last step's rows that crossed NVLink, max over ranks (from the all-gathered "
                        "counts); the dispatch stage time includes the counts all-gather and the layout kernel")

    # ---- roofline of the dominant kernel (GEMM1 + SwiGLU) and of dispatch ----
    peaks = load_peaks()
    # denominator: the burst bf16 peak for a sub-2-second timed region (the GPU stays near max
    # clock), the sustained one (measured back to back for 4 s under the power cap) for longer ones
    long_region = ms >= 2000.0
    bf16_peak = peaks["bf16_sus"] if long_region else peaks["bf16"]
    bf16_kind = (f"{'sustained' if long_region else 'burst'} ({peaks['src']}, MEASURED_PEAKS.json "
                 f"{'bf16_tflops_sustained' if long_region else 'bf16_tflops'}; timed region {ms / 1e3:.2f} s)")
    nf, nb = calls
    per = {k: v / max(nb if i >= 6 else nf, 1) for i, (k, v) in enumerate(stage_ms.items()) if (i < 6 or nb)}
    g1_flop = 2.0 * T * K * d * (2 * f)
    g2_flop = 2.0 * T * K * f * d
    g1_tf = g1_flop / (per["gemm1"] * 1e-3) / 1e12
    g2_tf = g2_flop / (per["gemm2"] * 1e-3) / 1e12
    disp_bytes = T * d * 2 + T * K * d * 2 + 8 * T * K
    comb_bytes = T * K * d * 2 + T * d * 2 + 8 * T * K
    disp_gbs = disp_bytes / (per["dispatch"] * 1e-3) / 1e9
    comb_gbs = comb_bytes / (per["combine"] * 1e-3) / 1e9
    esz = 1 if args.precision == "fp8" else 2
    nl = N // world
    w_bytes = nl * 3 * d * f * esz  # every local expert touched (checked below)
    g_ms = per["gemm1"] + per["gemm2"]
    stream_gbs = w_bytes / (g_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemm1_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(f"{T}x{d}x{N}x{K}x{f}" + ("-fp8" if args.precision == "fp8" else ""))

    if rank == 0:
        line = dict(
            metric=METRIC, value=value, unit="tokens/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
            ms_per_step=ms_step, higher_is_better=True,
            scaling="strong" if (cfg.get("train") and world > 1 and not args.tokens) else "weak", vs_baseline=None,
            dtype="bf16" if args.precision == "bf16" else "e4m3 (fp32 accumulate, bf16 activations in/out)",
            data="synthetic (device-generated reference-PRNG tokens and random-init weights)",
            config=dict(workload=cfg["workload"], T=T, d=d, n_experts=N, top_k=K, d_ff=f,
                        global_batch=T * world, parallelism=("ep%d (experts %d/rank; rows: %s)" % (world, N // world, transport))
                        if world > 1 else "single",
                        gemm_ctas=args.gemm_ctas or "auto",
                        l2=(f"inputs larger than L2 (x {T * d * 2 / 1e6:.0f} MB, weights "
                            f"{N // world * 3 * d * f * (1 if args.precision == 'fp8' else 2) / 1e9:.1f} GB per rank); "
                            "no flush needed")),
            roofline=(dict(bound="tensor", kernel="grouped GEMMs fwd+bwd (tcgen05, 6 launches)",
                           achieved=3 * (g1_flop + g2_flop) / (sum(per[k] for k in ("gemm1", "gemm2", "dgrad1_swiglu_bwd",
                                                                                      "dgrad2", "wgrad_out", "wgrad_in"))
                                                                * 1e-3) / 1e12,
                           peak=bf16_peak, unit="TFLOP/s", traffic=None, peak_kind=bf16_kind,
                           flop_per_step=3 * (g1_flop + g2_flop)) if train else
                      dict(bound="tensor", kernel="grouped GEMM1 + SwiGLU (tcgen05)", achieved=g1_tf,
                           peak=bf16_peak, unit="TFLOP/s", frac=g1_tf / bf16_peak,
                           frac_of_sustained=g1_tf / peaks["bf16_sus"], peak_kind=bf16_kind,
                           traffic=traffic, flop_per_launch=g1_flop, ms_per_launch=per["gemm1"])
                      if (args.precision == "bf16" and T * K >= 256 * nl * 4) else
                      dict(bound="tensor", kernel="grouped GEMM1 + SwiGLU (tcgen05 kind::f8f6f4, e4m3)", achieved=g1_tf,
                           peak=fp8_peak()[0], unit="TFLOP/s", frac=g1_tf / fp8_peak()[0],
                           peak_kind=fp8_peak()[1] + ": builder-measured denominator (no FP8 peak in "
                                                     "MEASURED_PEAKS.json)",
                           traffic=traffic, flop_per_launch=g1_flop, ms_per_launch=per["gemm1"])
                      if T * K >= 256 * nl * 4 else
                      dict(bound="hbm", kernel="grouped GEMM1+GEMM2 weight streaming (tcgen05)",
                           achieved=stream_gbs, peak=peaks["hbm"], unit="GB/s", frac=stream_gbs / peaks["hbm"],
                           traffic=None, bytes_per_launch=w_bytes, ms_per_launch=g_ms)),
            stages=dict(
                ms=per,
                gemm2=dict(achieved=g2_tf, unit="TFLOP/s", frac=g2_tf / (bf16_peak if args.precision == "bf16"
                                                                          else fp8_peak()[0])),
                dispatch=dict(achieved=disp_gbs, unit="GB/s", frac=disp_gbs / peaks["hbm"], bytes=disp_bytes),
                combine=dict(achieved=comb_gbs, unit="GB/s", frac=comb_gbs / peaks["hbm"], bytes=comb_bytes),
                layer_tflops=(g1_flop + g2_flop) / (ms_step * 1e-3) / 1e12),
            e2e=dict(value=e2e_val, unit="tokens/s", h2d_bytes_per_step=h2d_b, d2h_bytes_per_step=d2h_b,
                     steps=e2e_steps,
                     timing=("host wall clock: pinned H2D of x and dOut, forward_train + backward, D2H of out and "
                             "d_hidden, every step (copies double-buffered on two copy streams)" if train else
                             "host wall clock around `steps` pipelined cl_moe_forward_host_async calls (H2D of x "
                             "and D2H of out every call) + cl_moe_host_wait")),
            # ours per step, counted by CUPTI on an extra step (fallback: router, plan, dispatch,
            # GEMM1, GEMM2, combine (+ the EP peer layout kernel); training adds pad-plan and
            # combine-bwd, dgrad x2, dispatch-bwd, transposes x2, zero-pad x2, wgrad x2)
            gpu_launches=(per_step_launches if per_step_launches else
                          (17 if train else 6) + (1 if (world > 1 and "peer" in transport) else 0)) * args.steps,
            gpu_launches_source="counted (torch.profiler / CUPTI, kernels in namespace cmoe, one extra step)"
            if per_step_launches else "static per-step count",
            clocks=clocks,
        )
        if world > 1 and a2a is not None:
            line["a2a"] = a2a
        if not args.no_cpu_baseline and world == 1:
            t_s = pick_cpu_tokens(cfg)
            o, kind, inp, w_in, w_out = cpu_sample(cfg, t_s)
            jobs = os.cpu_count() or 1
            cpu_step(o, inp, w_in, w_out, K, jobs)  # warm
            t0 = time.perf_counter()
            cpu_step(o, inp, w_in, w_out, K, jobs)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = dict(
                value=t_s / dt, unit="tokens/s", cores=min(jobs, N), kind=kind, cpu_model=cpu_model(),
                host_threads=jobs,
                sample=f"{t_s} tokens of the same layer shape, one forward, fp32 (expert fan-out over "
                       f"{min(jobs, N)} threads)")
        if "frac" not in line["roofline"]:
            line["roofline"]["frac"] = line["roofline"]["achieved"] / line["roofline"]["peak"]
        if train:
            line["config"]["skew_gamma"] = cfg["skew"]
            line["config"]["mode"] = "forward_train + expert-FFN backward per step"
        print(json.dumps(line), flush=True)
    layer.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--gemm-ctas", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp8"])
    ap.add_argument("--tokens", type=int, default=0, help="override T (tokens per rank)")
    ap.add_argument("--ep-transport", default="peer", choices=["peer", "nccl"],
                    help="N>1 forward: rows over NVLink peer stores (dispatch kernel / GEMM2 epilogue) or NCCL p2p")
    ap.add_argument("--dry-run", action="store_true", help="rank plumbing only (gloo, no GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args.gpus))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.exit(f"--gpus {args.gpus} but the launcher started WORLD_SIZE={os.environ.get('WORLD_SIZE')} ranks")
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
