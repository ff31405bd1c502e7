#!/bin/bash
# Profiling recipe run on the GPU box (see /opt/skills/guides/B200_PROFILING.md).
#   1. launch list of one short bench run (gpu__time_duration per launch, cold & serialised)
#   2. one `ncu --set full` capture of the grouped GEMM kernels (GEMM1 and GEMM2 of one step)
# Each ncu pass runs only after the identical command exited 0 without ncu.
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_EXTRA}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_EXTRA}"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-grouped_gemm_kernel} -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-2} -o gpurun_out/prof_full $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done
