# (the SPO_CGROUP hook this drove was removed after the measurement; result in
# profiles/r01/v_groups.jsonl)
# VGL/VGH position groups on the line kernel (SPO_CGROUP=2: 2 positions per consumer
# warp, 8 warps) vs one position per warp (12 warps), k-power form, interleaved
for rep in 1 2; do for cg in 1 2; do
  SPO_CGROUP=$cg timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/cg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/cg.log').read().strip().splitlines()[-1]); print('cfg4 cgroup $cg', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  SPO_CGROUP=$cg timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/cg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/cg.log').read().strip().splitlines()[-1]); print('cfg3 cgroup $cg', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
done; done
