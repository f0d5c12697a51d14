# K1 A/B: limbs staged in the transform area (default, 3 CTAs/SM) vs + 4 CTAs/SM (k1m4) vs the previous layout (r4t320)
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "c1 or small_edge or medium or n1_2p14 or digest" > gpurun_out/tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tests.log
python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/ab_default.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab_default.log').read().strip().splitlines()[-1]); print('default', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items()})"
bash scripts/gpu_ab.sh k1m4 r4t320
