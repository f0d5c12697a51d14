# GPU parity tests then the bench (plain)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "stages", d["stages_ms"], "k2 frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"], "clk", d["clocks"])
PY
