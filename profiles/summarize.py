#!/usr/bin/env python3
"""Summarise ncu outputs brought back in gpurun_out/ into a committed markdown file.

    python profiles/summarize.py --tag r01_c2 [--launches gpurun_out/launches.csv]
                                 [--rep gpurun_out/prof_full.ncu-rep] [--bench gpurun_out/b.log]

Writes profiles/<tag>.md with (1) the per-kernel launch list (gpu__time_duration per launch,
cold and serialised under ncu: compare SHARES, not absolutes) and (2) the key `--set full`
metrics of the captured kernels (duration, DRAM bytes, tensor-pipe / FP64-pipe activity, SM
throughput, registers, occupancy) plus the bench line they belong to.
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % peak"),
    ("lts__t_sectors.sum", "L2 sectors"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster x"),
]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        if r[ui] == "ns":
            v /= 1e3
        elif r[ui] == "ms":
            v *= 1e3
        name = r[ki].split("(")[0]
        agg.setdefault(name, []).append(v)
    return agg


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = OrderedDict(kernel=r[h.index("Kernel Name")].split("(")[0])
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                d[label] = f"{r[i]} {u[i]}".strip()
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--rep", default=os.path.join(ROOT, "gpurun_out", "prof_full.ncu-rep"))
    ap.add_argument("--bench", default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    lines = [f"# ncu summary `{a.tag}`", ""]
    if a.note:
        lines += [a.note, ""]
    if a.bench and os.path.exists(a.bench):
        last = [ln for ln in open(a.bench).read().splitlines() if ln.startswith("{")][-1]
        j = json.loads(last)
        lines += ["## bench line (same build, no profiler)", "", "```json", json.dumps(j, indent=1), "```", ""]
    if os.path.exists(a.launches):
        agg = launch_table(a.launches)
        total = sum(sum(v) for k, v in agg.items() if not k.startswith("synth"))
        lines += ["## launch list (`--metrics gpu__time_duration.sum --clock-control none`)", "",
                  "cold-cache, serialised launches; compare shares, not absolutes", "",
                  "| kernel | launches | mean us | share of layer time |", "|---|---|---|---|"]
        for k, v in agg.items():
            share = "" if k.startswith("synth") else f"{100 * sum(v) / total:.1f} %"
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {share} |")
        lines.append("")
    if os.path.exists(a.rep):
        ms = full_metrics(a.rep)
        if ms:
            labels = list(ms[0].keys())
            lines += ["## `ncu --set full` (one launch each)", "", "| " + " | ".join(labels) + " |",
                      "|" + "---|" * len(labels)]
            for d in ms:
                lines.append("| " + " | ".join(str(d.get(k, "")) for k in labels) + " |")
            lines.append("")
    out = os.path.join(ROOT, "profiles", f"{a.tag}.md")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
