#!/bin/bash
# Profiling recipe (run under gpurun, one GPU):
#   bash profiles/ncu.sh <tag> [extra bench args]
# 1. the plain bench command (must exit 0 before any ncu pass),
# 2. the launch list of that same command (gpu__time_duration per launch),
# 3. one `ncu --set full` capture of the eval kernel on a one-chunk variant.
set -u
TAG=${1:-r01}
shift || true
mkdir -p gpurun_out
CMD="python bench.py $*"
SMALL="python bench.py --walkers 2048 --steps 1 --warmup 1 --no-cpu --no-e2e $*"
$CMD > gpurun_out/bench_${TAG}.log 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
$SMALL > gpurun_out/small_${TAG}.log 2>&1 || { echo "small bench failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:line_kernel|eval_tma_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} -f $SMALL > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "done"
