# quick A/B of library variants (paper_1402_5287_b200/lib/variants/libhk_<v>.so): stage times at C3
# usage: bash scripts/gpu_ab.sh v1 v2 ...   (env EXTRA="--config C4" to change the workload)
for v in "$@"; do
  HK_LIB_VARIANT=$PWD/paper_1402_5287_b200/lib/variants/libhk_$v.so python bench.py --no-cpu --no-e2e --steps 100 $EXTRA > gpurun_out/ab_$v.log 2>&1 || tail -3 gpurun_out/ab_$v.log
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items()}, 'warmA', round(d['warm_a']['ms_per_step'],4) if d.get('warm_a') else None)"
done
