# one rank's share of the strong-scaled config 4 job on ONE GPU (4096/N walkers), N = 1, 2, 4, 8:
# a projection of the walker-sharded run's per-rank time (no collective on that path), not a multi-GPU measurement
for w in 4096 2048 1024 512; do
  timeout 300 python bench.py --walkers $w --steps 10 --warmup 3 --no-cpu --no-e2e --no-extra 2> gpurun_out/rank_share_$w.err | tail -1
done > gpurun_out/rank_share.jsonl
