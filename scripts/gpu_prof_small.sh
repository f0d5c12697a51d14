# ncu --set full of K1/K2/K3 at the smaller BASELINE configs (C2, C5 Toeplitz, C5 circulant)
for C in C2 C5T C5C; do
  mkdir -p gpurun_out/$C
  CMD="python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu"
  for KRE in k1_slice k2_column k3_finish; do
    ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 3 -c 1 -f -o /tmp/prof_${C}_$KRE $CMD > gpurun_out/$C/ncu_$KRE.log 2>&1
    python scripts/ncu_summary.py /tmp/prof_${C}_$KRE.ncu-rep gpurun_out/$C/prof_$KRE.json > /dev/null
    python scripts/ncu_opcodes.py /tmp/prof_${C}_$KRE.ncu-rep "$KRE" > gpurun_out/$C/opcodes_$KRE.txt
    python scripts/ncu_lines.py /tmp/prof_${C}_$KRE.ncu-rep "$KRE" 30 > gpurun_out/$C/lines_$KRE.txt
  done
  python bench.py --config $C --steps 50 --no-e2e --no-cpu > gpurun_out/$C/bench.log 2>&1
done
true
