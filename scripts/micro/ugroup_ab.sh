# item order of the line kernel: unit-major (SPO_UGROUP=1, round-2 default) against groups of
# 4 / 8 / all units evaluated run-major (a run's records then come from L2 for all but the first unit)
timeout 1200 python scripts/micro/env_ab.py --envs "SPO_UGROUP=1;SPO_UGROUP=4;SPO_UGROUP=8;SPO_UGROUP=64" --cases cfg5-v,cfg5-v-2048w,cfg5-vgh-2048w,cfg4-vgh-2048w,cfg4-vgh-512w,cfg4-v-4096w,cfg3-vgl-1024w,cfg2-v 2>&1 | grep '^{'
for ug in 1 8 64 1 8 64; do
  SPO_UGROUP=$ug timeout 600 python bench.py --config 5 --no-e2e --no-cpu --steps 5 2>/dev/null | python -c "
import sys,json
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('cfg5 ugroup $ug', '%.4g'%d['value'], '%.2f ms/step'%d['ms_per_step'], 'V launch %.2f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
