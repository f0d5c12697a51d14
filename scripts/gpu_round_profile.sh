# Round evidence: full bench line, ncu launch list of the same command, ncu --set full summaries
# of K1/K2/K3 (json + source-line and opcode breakdowns).  Outputs in gpurun_out/.
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
KRES="k1_slice k2_column k3_finish" PHASES="" bash scripts/gpu_prof_k.sh
