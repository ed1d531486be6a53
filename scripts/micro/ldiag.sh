# (the SPO_LDIAG / SPO_UGROUP hooks this drove were removed from spo_eval_line.cu after the
# measurement; results in profiles/r01/line_energy_diag.txt)
# line-kernel energy diagnostics (wrong results by design): SPO_LDIAG=1 drops the
# output stores, =2 contracts only the first of each position's four planes
for d in 0 1 2 3 0; do SPO_LDIAG=$d python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ld.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ld.log').read().strip().splitlines()[-1]); print('diag $d', '%.4g'%d['value'], '%.3f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['clocks']['reasons'])"; done
