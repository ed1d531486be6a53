# (the 1024-byte-unit build this drove was removed after the measurement: 29% slower on
# config 4, 22% on config 3; see DESIGN)
# line kernel with 1024-byte units (8 fp32 orbitals per consumer thread, 12 ring slots
# of 16 KB, 8 consumer warps at 232 registers: more ILP per warp, per-position work
# amortised over twice the lanes) against the default; variant build via SPO_LIB
P=$PWD/paper_1611_02665_b200
for v in w8; do SPO_LIB=$P/libspo_b200_$v.so timeout 300 python scripts/stress_line.py 150 8 | tail -1; done
for rep in 1 2; do for v in default w8; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  timeout 180 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/w8.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/w8.log').read().strip().splitlines()[-1]); print('cfg4 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  timeout 180 python bench.py --config 3 --no-cpu --no-e2e --steps 20 > gpurun_out/w8.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/w8.log').read().strip().splitlines()[-1]); print('cfg3 $v', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done
unset SPO_LIB
