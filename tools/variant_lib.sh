#!/bin/bash
# Build a variant of the library with extra nvcc flags for tc_pass.cu only
# (A/B experiments): tools/variant_lib.sh NAME "-DFOO=1 ..." -> oldlib/NAME.so
set -e
NAME=$1; shift
FLAGS="$*"
CS=paper_1505_04650_b200/csrc
mkdir -p oldlib/obj_$NAME
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr $FLAGS -c $CS/tc_pass.cu -o oldlib/obj_$NAME/tc_pass.o
OBJS=$(ls $CS/build/*.o | grep -v tc_pass.o | grep -v tc_debug.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o oldlib/$NAME.so $OBJS oldlib/obj_$NAME/tc_pass.o -cudart static
echo oldlib/$NAME.so
