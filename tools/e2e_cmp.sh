# cfg2 device and end-to-end times over repeated runs (host-path A/B checks)
for t in 1 2 3 4; do
  python bench.py --no-cpu --no-extra --steps 40 > gpurun_out/b$t.json 2>/dev/null
  python -c "
import json; l=json.loads(open('gpurun_out/b$t.json').read().strip().splitlines()[-1]); print('run $t', round(l['ms_per_step'],4), round(l['e2e']['ms'],4))"
done
