# line kernel positions per run (BPL) and ring slots: variant libraries built with
# scripts/micro/build_variant.py, loaded through SPO_LIB; stress-checked, then
# config 4 (VGH, k-power) and config 3 (VGL) interleaved
P=paper_1611_02665_b200
for v in bpl32 bpl96 bpl128; do SPO_LIB=$PWD/$P/libspo_b200_$v.so timeout 300 python scripts/stress_line.py 120 5 | tail -1; done
for rep in 1 2; do for v in default bpl32 bpl96 bpl128; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$PWD/$P/libspo_b200_$v.so; fi
  timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bp.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1]); print('cfg4 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/bp.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1]); print('cfg3 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done
unset SPO_LIB
