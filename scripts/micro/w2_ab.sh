# (the 256-byte-unit build defines this drove were removed after the measurement:
# 16 warps x 2 orbitals per thread 32% slower, 12 warps 14% slower; see DESIGN)
# line kernel with 256-byte units (2 fp32 orbitals per consumer thread, 48 slots of
# 4 KB): 16 consumer warps at 112 registers (w2) or 12 at 160 (w2x12), against the
# default 512-byte units (12 warps); variant builds via SPO_LIB, stress-checked first
P=$PWD/paper_1611_02665_b200
for v in w2 w2x12; do SPO_LIB=$P/libspo_b200_$v.so timeout 300 python scripts/stress_line.py 150 8 | tail -1; done
for rep in 1 2; do for v in default w2 w2x12; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/w2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/w2.log').read().strip().splitlines()[-1]); print('cfg4 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/w2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/w2.log').read().strip().splitlines()[-1]); print('cfg3 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done
unset SPO_LIB
