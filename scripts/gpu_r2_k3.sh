# round-2: smoke + parity suite + K3 ncu capture
set -u
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --maxfail=15 -p no:cacheprovider > gpurun_out/tests.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/tests.log
KRES="k3_finish" PHASES="" bash scripts/gpu_prof_k.sh
cat gpurun_out/plain_small.log | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['stages_ms'], d['value'])"
