# quick A/B of bench configurations (no tests)
for v in 0 1; do
  HK_K2_DIAG=$v python bench.py --no-cpu --no-e2e --steps 200 > gpurun_out/ab.log 2>&1 || tail -3 gpurun_out/ab.log
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('diag=$v', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()})"
done
