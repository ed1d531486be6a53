# fp32 z-second-derivative through the (ax ay)-weighted z rows (312 FMAs per
# VGH orbital instead of 328; VGL 284 instead of 300) against the previous
# contraction (libspo_b200_old.so), interleaved on one box
P=$PWD/paper_1611_02665_b200
for rep in 1 2; do for v in default z2; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  timeout 180 python bench.py --no-cpu --no-e2e --no-extra --steps 10 > gpurun_out/z2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/z2.log').read().strip().splitlines()[-1]); print('cfg4 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
  timeout 180 python bench.py --config 3 --no-cpu --no-e2e --no-extra --steps 20 > gpurun_out/z2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/z2.log').read().strip().splitlines()[-1]); print('cfg3 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
  timeout 180 python bench.py --config 2 --no-cpu --no-e2e --no-extra --steps 50 > gpurun_out/z2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/z2.log').read().strip().splitlines()[-1]); print('cfg2 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
done; done
unset SPO_LIB
