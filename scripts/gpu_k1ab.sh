# K1 A/B (variants under paper_1402_5287_b200/lib/variants) + parity of the candidate variant
CAND=${CAND:-both}
HK_LIB_VARIANT=$PWD/paper_1402_5287_b200/lib/variants/libhk_$CAND.so timeout 900 python -m pytest tests -m gpu -x -q -k "not C4" > gpurun_out/tests_$CAND.log 2>&1; echo "pytest($CAND) rc=$?"; tail -2 gpurun_out/tests_$CAND.log
for r in 1 2; do bash scripts/gpu_ab.sh "$@"; done
