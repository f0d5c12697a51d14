# bench line for every BASELINE config (device-resident, no e2e / cpu legs)
for c in C1 C2 C3 C4 C5T C5C; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --steps 50 > gpurun_out/cfg_$c.log 2>&1 || { echo "$c failed"; tail -3 gpurun_out/cfg_$c.log; continue; }
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/cfg_{c}.log").read().strip().splitlines()[-1])
r = d["roofline"]
print(c, "ms %.4f" % d["ms_per_step"], "mv/s %.0f" % d["value"], {k: round(v, 4) for k, v in d["stages_ms"].items()},
      "step_frac %.3f" % r["step_frac"], "K2 frac %.3f" % r["frac"], "warmA %.0f" % d["warm_a"]["value"],
      "tp %.0f" % d["throughput"]["value"], "fp64 %.3f ms" % d["fp64_fft"]["ms_per_step"])
PY
done
