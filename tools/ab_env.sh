#!/bin/bash
# Same-box A/B of environment settings on the bench (run on the GPU box from the repo root):
#   tools/ab_env.sh "<bench args>" "<envA>" "<envB>" ... ; each setting runs ROUNDS times, interleaved.
# Prints one line per run: setting, step ms, per-stage ms (router/dispatch/gemm1/gemm2/combine), SM clock.
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
print(f"{s:45s} step {d['ms_per_step']:.3f} ms  tok/s {d['value']/1e6:.3f}M  r {st['router']:.3f} d {st['dispatch']:.3f} "
      f"g1 {st['gemm1']:.3f} g2 {st['gemm2']:.3f} c {st['combine']:.3f}  sm {d['clocks'].get('sm_mhz')} e2e {d['e2e']['value']/1e6:.3f}M")
PY
  done
done
