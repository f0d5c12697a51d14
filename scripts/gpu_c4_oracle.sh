# C4 oracle digests on the GPU box's host cores (scripts/oracle_digests.py --dig-dir; the GPU idles).
# Chunks 0..103 of 128 (128 rows each) here; the top chunks run in the CPU container.
mkdir -p gpurun_out/C4_dig
echo "nproc $(nproc)"
timeout ${C4_SECONDS:-5400} python scripts/oracle_digests.py C4 --chunks ${C4_CHUNKS:-0:104} \
  --dig-dir gpurun_out/C4_dig --threads $(nproc) --no-assemble > gpurun_out/c4_box.log 2>&1
echo "oracle rc=$?"; tail -2 gpurun_out/c4_box.log; ls gpurun_out/C4_dig | wc -l
