# A/B of library variants over several configs: CONFIGS="C2 C5T" bash scripts/gpu_ab_configs.sh v1 v2 ...
for C in ${CONFIGS:-C2 C5T C5C C3}; do
  echo "== $C"
  EXTRA="--config $C" bash scripts/gpu_ab.sh "$@"
done
