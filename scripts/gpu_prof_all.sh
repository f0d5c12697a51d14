# launch list + one full ncu capture per hot kernel (k1, k2, k3a, k3b)
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_slice|k2_column|k3a_row|k3b_carry" -s 4 -c 4 -o gpurun_out/prof_all -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
