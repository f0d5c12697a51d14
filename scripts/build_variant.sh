#!/bin/bash
# dev A/B: build libhk with extra -D flags into paper_1402_5287_b200/lib/variants/libhk_<name>.so
# usage: scripts/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1402_5287_b200/lib/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared --expt-relaxed-constexpr $2 -I include \
  -o paper_1402_5287_b200/lib/variants/libhk_$1.so paper_1402_5287_b200/csrc/*.cu
echo "built $1"
