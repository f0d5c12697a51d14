set -x
python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_c3.log
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_column -s 1 -c 1 -o gpurun_out/prof_k2 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
ls -la gpurun_out
