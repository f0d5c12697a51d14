# GPU parity tests (fast subset unless FULL=1) + bench stage times
if [ "$FULL" = 1 ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "pytest rc=$?"
else timeout 900 python -m pytest tests -m gpu -x -q -k "not C4" > gpurun_out/tests.log 2>&1; echo "pytest rc=$?"; fi
tail -15 gpurun_out/tests.log | grep -E "passed|failed|Error|error|assert" | head -20
python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['value'],1), {k: round(x,4) for k,x in d['stages_ms'].items()}, 'warmA', round(d['warm_a']['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"
