# ncu --set full capture of kernels matching each regex in $KRES (one launch each) during a short
# bench; summaries (json, top source lines, opcode mix) written to gpurun_out/, reports deleted
# unless KEEP=1 (they exceed gpurun's copy-back limit).
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu $EXTRA"
$CMD > gpurun_out/plain_small.log 2>&1 || { echo plain failed; tail gpurun_out/plain_small.log; exit 1; }
for KRE in $KRES; do
  ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${SKIP:-3} -c 1 -f -o /tmp/prof_$KRE $CMD > gpurun_out/ncu_full_$KRE.log 2>&1
  echo "ncu $KRE rc=$?"
  python scripts/ncu_summary.py /tmp/prof_$KRE.ncu-rep gpurun_out/prof_$KRE.json > /dev/null
  python scripts/ncu_lines.py /tmp/prof_$KRE.ncu-rep "$KRE" 45 > gpurun_out/lines_$KRE.txt
  python scripts/ncu_opcodes.py /tmp/prof_$KRE.ncu-rep "$KRE" > gpurun_out/opcodes_$KRE.txt
  [ -n "$PHASES" ] && python scripts/ncu_phases.py /tmp/prof_$KRE.ncu-rep "$KRE" $PHASES > gpurun_out/phases_$KRE.txt
  if [ "$KEEP" = 1 ]; then cp /tmp/prof_$KRE.ncu-rep gpurun_out/; fi
done
true
