for v in 0 256 512; do
  ODX_RES_LAT=$v python bench.py --workload cfg1 --no-cpu --no-extra --steps 20 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lat $v', round(l['ms_per_step'],4), l['final_status'])"
done
