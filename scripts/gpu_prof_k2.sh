CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_column -s 1 -c 1 -o gpurun_out/prof_k2 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
