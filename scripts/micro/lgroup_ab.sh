# (the SPO_LGROUP hook this drove was removed after the measurement; result in
# profiles/r01/v_groups.jsonl)
# VGL position pairs at 12 warps (SPO_LGROUP=2, k-power form) vs one position per warp,
# interleaved: config 3 (VGL, 1.19 positions per cell) and a 2/cell VGL batch
for rep in 1 2; do for lg in 1 2; do
  SPO_LGROUP=$lg timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/lg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/lg.log').read().strip().splitlines()[-1]); print('cfg3 lgroup $lg', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
  SPO_LGROUP=$lg timeout 180 python bench.py --config 4 --kind vgl --no-cpu --no-e2e --steps 10 > gpurun_out/lg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/lg.log').read().strip().splitlines()[-1]); print('cfg4-vgl lgroup $lg', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
done; done
