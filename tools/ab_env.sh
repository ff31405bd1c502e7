#!/bin/bash
# Same-box A/B of environment settings on the bench (run on the GPU box from the repo root):
#   tools/ab_env.sh "<bench args>" "<envA>" "<envB>" ... ; each setting runs ROUNDS times, interleaved.
# Prints one line per run: setting, step ms, every per-stage ms the bench reports, SM clock.
args="$1"; shift
ROUNDS=${ROUNDS:-2}
for r in $(seq $ROUNDS); do
  for setting in "$@"; do
    out=$(env $setting python bench.py $args --no-cpu-baseline 2>/dev/null | tail -1)
    python3 - "$setting" "$out" <<'PY'
import json, sys
s, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
except Exception:
    print(s, "FAILED", line[:200]); sys.exit()
st = d["stages"]["ms"]
short = {"router": "r", "dispatch": "d", "gemm1": "g1", "gemm2": "g2", "combine": "c", "combine_bwd": "cb",
         "dgrad1_swiglu_bwd": "dg1", "dgrad2": "dg2", "dispatch_bwd": "db", "transposes": "tr",
         "wgrad_out": "wo", "wgrad_in": "wi"}
stages = " ".join(f"{short.get(k, k)} {v:.3f}" for k, v in st.items() if k != "plan")
print(f"{s:45s} step {d['ms_per_step']:.3f} ms  tok/s {d['value']/1e6:.3f}M  {stages}  "
      f"sm {d['clocks'].get('sm_mhz')} e2e {d['e2e']['value']/1e6:.3f}M")
PY
  done
done
