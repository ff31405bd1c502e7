#!/bin/bash
# DRAM bytes and (serialised, cold-cache) duration of one step's grouped GEMMs under several
# tile-order / cache-hint settings (the knobs of launch_gemm, host_forward.cuh). Run on the GPU box:
#   tools/gemm_dram_sweep.sh <config> <gemms per step> "<env setting>" ...
cfg=$1; n=$2; shift 2
mkdir -p gpurun_out/gemm_dram
for setting in "$@"; do
  tag=${cfg}_$(echo $setting | tr '= ' '__')
  env $setting timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:grouped_gemm --launch-skip $((3 * n)) --launch-count $n --csv --log-file gpurun_out/gemm_dram/$tag.csv \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/gemm_dram/$tag.log 2>&1
  echo "== $setting"
  python3 - gpurun_out/gemm_dram/$tag.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; data = rows[1:]
ik = hdr.index("Kernel Name"); im = hdr.index("Metric Name"); iv = hdr.index("Metric Value"); iid = hdr.index("ID")
out = {}
for r in data:
    out.setdefault(r[iid], [r[ik][:48]]).append((r[im], r[iv]))
for k, v in out.items():
    d = dict(v[1:])
    print(k, v[0], "rd %.1f GB wr %.1f GB t %.2f ms" % (float(d["dram__bytes_read.sum"].replace(",", "")) / 1e9 if "dram__bytes_read.sum" in d else -1,
          float(d["dram__bytes_write.sum"].replace(",", "")) / 1e9 if "dram__bytes_write.sum" in d else -1,
          float(d["gpu__time_duration.sum"].replace(",", "")) / 1e6))
PY
done
