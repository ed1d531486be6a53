# line kernel: positions taken from a shared per-run counter (SPO_DYNAMIC=1) vs the
# rotated static assignment (SPO_DYNAMIC=0), interleaved; config 4 VGH (k-power), config 3 VGL,
# config 4 on the B-spline form
for rep in 1 2; do for ro in 0 1; do
  SPO_DYNAMIC=$ro timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ro.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ro.log').read().strip().splitlines()[-1]); print('cfg4 dynamic $ro', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  SPO_DYNAMIC=$ro timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/ro.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ro.log').read().strip().splitlines()[-1]); print('cfg3 dynamic $ro', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  SPO_DYNAMIC=$ro timeout 180 python bench.py --no-cpu --no-e2e --steps 10 --form bspline > gpurun_out/ro.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ro.log').read().strip().splitlines()[-1]); print('cfg4 bspline dynamic $ro', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done
