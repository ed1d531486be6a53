# interleaved bench A/B of experiment builds: bash scripts/micro/variant_ab.sh default v1 v2 ...
P=$PWD/paper_1611_02665_b200
for rep in 1 2; do for v in "$@"; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  for c in 4 3; do
    timeout 180 python bench.py --config $c --no-cpu --no-e2e --no-extra --steps 10 > gpurun_out/vab.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/vab.log').read().strip().splitlines()[-1]); print('cfg$c $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['config']['path'])"
  done
done; done
unset SPO_LIB
