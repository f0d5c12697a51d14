# round-2 K3 A/B + gpu tests (default build = 2-row/160-thread K3)
set -u
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_digests.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/tests.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/tests.log
python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/ab_default.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab_default.log').read().strip().splitlines()[-1]); print('default', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items()})"
bash scripts/gpu_ab.sh r4t320
