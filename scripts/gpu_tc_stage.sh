# F4: tcgen05 kind::i8 radix-32 NTT stage vs the radix-2 ALU stage (scripts/tc_ntt_stage.cu)
set -u
timeout 120 ./scripts/tc_ntt_stage 4000 > gpurun_out/tc_stage.log 2>&1; echo "tc_stage rc=$?"; cat gpurun_out/tc_stage.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tc_stage|alu_stage" -s 2 -c 4 -f -o /tmp/tc_prof ./scripts/tc_ntt_stage 400 > gpurun_out/tc_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/tc_prof.ncu-rep gpurun_out/tc_stage_ncu.json > /dev/null 2>&1; echo "summary rc=$?"
python scripts/ncu_opcodes.py /tmp/tc_prof.ncu-rep tc_stage > gpurun_out/tc_stage_opcodes.txt 2>&1
python scripts/ncu_opcodes.py /tmp/tc_prof.ncu-rep alu_stage > gpurun_out/alu_stage_opcodes.txt 2>&1
true
