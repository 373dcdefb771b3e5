for t in 4 8 4 8; do
  ODX_HOST_THREADS=$t python bench.py --no-cpu --no-extra --steps 40 > gpurun_out/b$t.json 2>/dev/null
  python -c "
import json; l=json.loads(open('gpurun_out/b$t.json').read().strip().splitlines()[-1]); print('threads $t', round(l['ms_per_step'],4), round(l['e2e']['ms'],4), round(l['e2e_policy_guess']['ms'],4))"
done
