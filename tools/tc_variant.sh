#!/bin/bash
# Build pass_tc ring-depth variants: tools/tc_variant_ST_SSP_AST.bin
set -e
cd "$(dirname "$0")/.."
C=paper_1505_04650_b200/csrc
for v in "$@"; do
  IFS=_ read st ssp ast x <<< "$v"
  x=${x:-0}
  /usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
    -DCNMF_TC_RINGS -DCNMF_TC_ST=$st -DCNMF_TC_SSP=$ssp -DCNMF_TC_AST=$ast -DCNMF_X=$x \
    tools/tc_variant.cu $C/common.cu -o tools/tc_variant_$v.bin -lcuda 2>&1 | grep -i error || true &
done
wait
