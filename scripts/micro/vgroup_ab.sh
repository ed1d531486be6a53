# V position groups: branch-free loop when the group's positions share one cell
# (config 5's fp64 V at 16/cell, fp32 V at 4/cell) vs the previous build
P=$PWD/paper_1611_02665_b200
for rep in 1 2; do for v in default prev; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  timeout 300 python bench.py --config 5 --steps 3 --no-cpu --no-e2e --no-extra > gpurun_out/vg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/vg.log').read().strip().splitlines()[-1]); print('cfg5 $v', '%.4g'%d['value'], '%.3f'%d['ms_per_step'], 'V launch %.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  timeout 300 python bench.py --config 4 --kind v --chunk 1048576 --steps 10 --no-cpu --no-e2e --no-extra > gpurun_out/vg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/vg.log').read().strip().splitlines()[-1]); print('cfg4-V4 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
done; done
unset SPO_LIB
