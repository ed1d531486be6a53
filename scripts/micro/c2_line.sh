# config 2 VGH (0.15 positions per cell): per-position TMA kernel vs line kernel, both forms
for rep in 1 2; do for f in bspline kpower; do for ln in 0 1; do
  SPO_LINE=$ln timeout 120 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu --no-e2e --form $f > gpurun_out/c2l.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/c2l.log').read().strip().splitlines()[-1]); print('$f line=$ln', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], d['config']['path'])"
done; done; done
