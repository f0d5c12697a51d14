# A/B of library variants: warm-A, throughput and step for one config, repeated
C=${C:-C1}
for r in 1 2 3; do for v in "$@"; do
  HK_LIB_VARIANT=$PWD/paper_1402_5287_b200/lib/variants/libhk_$v.so python bench.py --config $C --no-cpu --no-e2e --steps 100 > gpurun_out/abf_$v.log 2>&1 || tail -3 gpurun_out/abf_$v.log
  python -c "
import json; d=json.loads(open('gpurun_out/abf_$v.log').read().strip().splitlines()[-1]); print('$v', '$C', 'step', round(d['ms_per_step'],4), 'warmA', round(d['warm_a']['ms_per_step'],4), 'tp', round(d['throughput']['ms_per_matvec'],4))"
done; done
