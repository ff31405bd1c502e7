#!/bin/bash
# Round bench sweep on one B200 (run under gpurun from the repo root). Lines land in
# gpurun_out/bench/<name>.log; copy the ones to keep into profiles/bench_r01/.
mkdir -p gpurun_out/bench
run() { name=$1; shift; python bench.py "$@" > gpurun_out/bench/$name.log 2> gpurun_out/bench/$name.err; echo "$name rc=$?"; }
run r01_c2_bf16 --config c2
run r01_c2_fp8 --config c2 --precision fp8
run r01_c1 --config c1
run r01_c3 --config c3
for t in 64 128 256 512; do
  run r01_c4_bf16_T$t --config c4 --tokens $t
  run r01_c4_fp8_T$t --config c4 --tokens $t --precision fp8
done
run r01_c5 --config c5
run r01_ref --impl reference --steps 3 --warmup 1
