#!/bin/bash
# Profiling recipe run on the GPU box (see /opt/skills/guides/B200_PROFILING.md).
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 6 -c 2 -o gpurun_out/prof_gemm $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done
