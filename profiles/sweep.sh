#!/bin/bash
# Parameter sweep helper (run under gpurun): bash profiles/sweep.sh <tag> "<env assignments>" ...
TAG=$1; shift
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  BENCH_ARGS=$(echo "$spec" | grep -o -- "--.*")
  spec=$(echo "$spec" | sed "s/--.*//")
  i=$((i+1))
  env $spec timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e $BENCH_ARGS > gpurun_out/sw_${TAG}_$i.log 2>&1
  echo "$spec" >> gpurun_out/sw_${TAG}_$i.log
done
