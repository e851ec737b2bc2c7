#!/bin/bash
# Build the pass_tc timeline tracer against the library's common.cu.
set -e
cd "$(dirname "$0")/.."
C=paper_1505_04650_b200/csrc
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
  tools/tc_trace.cu $C/common.cu -o tools/tc_trace.bin -lcuda
