# dev A/B of library variants by stage times (scripts/stage_times.py); usage: bash scripts/gpu_stage_ab.sh CFG v1 v2 ...
cfg=$1; shift
python scripts/stage_times.py $cfg
for v in "$@"; do
  HK_LIB_VARIANT=$PWD/paper_1402_5287_b200/lib/variants/libhk_$v.so python scripts/stage_times.py $cfg || echo "$v failed"
done
