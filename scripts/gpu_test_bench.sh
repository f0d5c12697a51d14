# GPU parity tests then the bench (plain)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/tests.log
python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print("warm", round(d["warm_a"]["value"],1) if d.get("warm_a") else None, "value", round(d["value"],1), "ms", round(d["ms_per_step"],4), "stages", {k: round(v,4) for k,v in d["stages_ms"].items()}, "k2 frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"],1), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
