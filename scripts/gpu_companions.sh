# Companion-kernel evidence (A5/A6): event times + work rates, then ncu --set full of k6_schoolbook and
# k5_leaf at C1 (n = 64, P = 3328) and n = 128, P = 33,216; summaries to gpurun_out/.
python scripts/companions_profile.py > gpurun_out/companions.log 2>&1; echo "companions rc=$?"
for CASE in 64:3328 128:33216; do
  for K in k6_schoolbook k5_leaf; do
    T=${K}_${CASE/:/_}
    ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c 1 -f -o /tmp/prof_$T \
      python scripts/companions_profile.py --cases $CASE > gpurun_out/ncu_$T.log 2>&1
    echo "ncu $T rc=$?"
    python scripts/ncu_summary.py /tmp/prof_$T.ncu-rep gpurun_out/prof_$T.json > /dev/null
    python scripts/ncu_opcodes.py /tmp/prof_$T.ncu-rep "$K" > gpurun_out/opcodes_$T.txt
  done
done
true
