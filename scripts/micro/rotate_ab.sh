# line kernel: rotating the run's positions over the consumer warps (default) vs a
# fixed assignment (SPO_ROTATE=0), interleaved; config 4 VGH (k-power), config 3 VGL,
# config 4 on the B-spline form
for rep in 1 2; do for ro in 0 1; do
  SPO_ROTATE=$ro timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ro.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ro.log').read().strip().splitlines()[-1]); print('cfg4 rotate $ro', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  SPO_ROTATE=$ro timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/ro.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ro.log').read().strip().splitlines()[-1]); print('cfg3 rotate $ro', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  SPO_ROTATE=$ro timeout 180 python bench.py --no-cpu --no-e2e --steps 10 --form bspline > gpurun_out/ro.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ro.log').read().strip().splitlines()[-1]); print('cfg4 bspline rotate $ro', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done
