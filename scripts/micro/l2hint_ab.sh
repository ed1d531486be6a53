# result (one box): no difference -- config 4 7.74e10 either way, config 3 8.93-9.00e10
# L2 evict_last policy on the line kernel's plane loads (default) vs evict_normal
# (SPO_L2HINT=0), k-power form, config 4 and config 3, interleaved
for rep in 1 2; do for h in 1 0; do
  SPO_L2HINT=$h timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/l2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/l2.log').read().strip().splitlines()[-1]); print('cfg4 hint $h', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  SPO_L2HINT=$h timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/l2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/l2.log').read().strip().splitlines()[-1]); print('cfg3 hint $h', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done
