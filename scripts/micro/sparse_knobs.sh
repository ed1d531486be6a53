# per-position TMA kernel knobs on config 2 (sparse VGH, 16,384 positions; V, 98,304):
# chunk width SPO_CW (elements) x item size SPO_BP (positions), bench.py --config 2 steps
for cw in 0 64 32; do for bp in 0 1 2 4 8; do
  if [ $bp = 0 ]; then unset SPO_BP; else export SPO_BP=$bp; fi
  if [ $cw = 0 ]; then unset SPO_CW; else export SPO_CW=$cw; fi
  timeout 120 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/sk.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/sk.log').read().strip().splitlines()[-1]); print('cw $cw bp $bp', '%.4g'%d['value'], '%.4f'%d['ms_per_step'])"
done; done
