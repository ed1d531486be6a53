# (the SPO_LDIAG / SPO_UGROUP hooks this drove were removed from spo_eval_line.cu after the
# measurement; results in profiles/r01/line_energy_diag.txt)
# line kernel: units per ticket group (SPO_UGROUP), interleaved repeats
for g in 1 2 4 8 1 2 4; do SPO_UGROUP=$g python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ug.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ug.log').read().strip().splitlines()[-1]); print('ugroup $g', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"; done
