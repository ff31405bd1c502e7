#!/bin/bash
# compute-sanitizer over the hot-path kernels at small shapes (run on the GPU box from the repo
# root; logs into gpurun_out/sanitizer/). memcheck + synccheck over everything; racecheck
# (shared-memory hazards) per kernel family, each router variant forced in its own process.
out=gpurun_out/sanitizer
mkdir -p $out
CS="timeout 900 compute-sanitizer"
$CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_run.py all > $out/memcheck.log 2>&1; echo "memcheck rc=$?" >> $out/summary.txt
$CS --tool synccheck --error-exitcode 9 python tools/sanitize_run.py all > $out/synccheck.log 2>&1; echo "synccheck rc=$?" >> $out/summary.txt
for v in ws lat small big; do
  CL_MOE_ROUTER=$v $CS --tool racecheck --racecheck-report all --error-exitcode 9 -k regex:router python tools/sanitize_run.py fwd > $out/racecheck_router_$v.log 2>&1
  echo "racecheck router=$v rc=$?" >> $out/summary.txt
done
$CS --tool racecheck --racecheck-report all --error-exitcode 9 -k regex:"dispatch|combine|plan" python tools/sanitize_run.py all > $out/racecheck_dispatch_combine_plan.log 2>&1; echo "racecheck dispatch/combine/plan rc=$?" >> $out/summary.txt
$CS --tool racecheck --racecheck-report all --error-exitcode 9 -k regex:grouped_gemm python tools/sanitize_run.py fwd > $out/racecheck_gemm.log 2>&1; echo "racecheck grouped_gemm rc=$?" >> $out/summary.txt
cat $out/summary.txt
