# (the SPO_RING hook and the general issue cursor it selected were removed after the
# measurement: 8 warps x 3 stages ran 16% slower than 12 x 2 on config 2; see DESIGN)
# per-position TMA kernel: 12 warps x 2-stage ring (default) vs 8 warps x 3 stages
# (SPO_RING=3), config 2 VGH / V and a 64^3 N=4096 0.25-per-cell VGH batch, interleaved
for rep in 1 2; do for rg in 2 3; do
  SPO_RING=$rg timeout 120 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/rg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/rg.log').read().strip().splitlines()[-1]); print('cfg2 vgh ring $rg', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], d['config']['path'])"
  SPO_RING=$rg timeout 120 python bench.py --config 2 --kind v --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/rg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/rg.log').read().strip().splitlines()[-1]); print('cfg2 v ring $rg', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], d['config']['path'])"
done; done
