# (measured with an Estrin-form build as the default and the Horner form as the variant;
# Estrin was reverted: config 4 +0.1%, config 3 -2.7%)
# k-power z-sums: Estrin form (6 FMAs, depth 2; current) vs the Horner form (7 ops, depth 5;
# variant library libspo_b200_horner.so via SPO_LIB), interleaved
P=$PWD/paper_1611_02665_b200
for rep in 1 2; do for v in horner estrin; do
  if [ $v = estrin ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_horner.so; fi
  timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/es.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/es.log').read().strip().splitlines()[-1]); print('cfg4 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/es.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/es.log').read().strip().splitlines()[-1]); print('cfg3 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done
unset SPO_LIB
