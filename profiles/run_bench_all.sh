#!/bin/bash
# Round bench sweep on one B200 (run under gpurun from the repo root). Lines land in
# gpurun_out/bench/<round>_<name>.log; copy the ones to keep into profiles/bench_<round>/.
R=${ROUND:-r02}
mkdir -p gpurun_out/bench
run() { name=${R}_$1; shift; python bench.py "$@" > gpurun_out/bench/$name.log 2> gpurun_out/bench/$name.err; echo "$name rc=$?"; }
run c2_bf16 --config c2
run c2_fp8 --config c2 --precision fp8
run c1 --config c1
run c3 --config c3
for t in 64 128 256 512; do
  run c4_bf16_T$t --config c4 --tokens $t
  run c4_fp8_T$t --config c4 --tokens $t --precision fp8
done
run c5 --config c5
run ref --impl reference --steps 3 --warmup 1
