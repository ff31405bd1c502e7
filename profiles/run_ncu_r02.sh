#!/bin/bash
# Round-2 ncu recipe (one GPU; each ncu pass only after the same command exited 0 without ncu):
#   1. launch list of the headline command (gpu__time_duration per launch, cold and serialised)
#   2. --set full of one GEMM1 + one GEMM2 launch of a C2 bf16 step
#   3. --set full of the router (DMMA + finish) / plan / dispatch / combine of one C2 step
#   4. --set full of one FP8 GEMM1 + GEMM2
set -x
mkdir -p gpurun_out/ncu
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_c2.csv $CMD > gpurun_out/ncu/launch.log 2>&1
CMD1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD1 > gpurun_out/ncu/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 6 -c 2 -o gpurun_out/ncu/r02_c2_gemms $CMD1 > gpurun_out/ncu/gemms.log 2>&1
ncu --set full --clock-control none -k regex:"router|plan|dispatch|combine" -s 15 -c 5 -o gpurun_out/ncu/r02_c2_small $CMD1 > gpurun_out/ncu/small.log 2>&1
CMD8="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --precision fp8"
$CMD8 > gpurun_out/ncu/plain8.log 2>&1 && \
ncu --set full --clock-control none -k regex:grouped_gemm_kernel -s 8 -c 2 -o gpurun_out/ncu/r02_c2_fp8_gemms $CMD8 > gpurun_out/ncu/fp8.log 2>&1
echo done
