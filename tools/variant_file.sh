#!/bin/bash
# Build a library variant with extra nvcc flags for ONE source file (A/B and
# trace builds): tools/variant_file.sh NAME FILE.cu "-DFOO ..." -> varlibs/NAME.so
set -e
NAME=$1; FILE=$2; shift 2
FLAGS="$*"
CS=paper_1505_04650_b200/csrc
mkdir -p varlibs/obj_$NAME
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr $FLAGS -c $CS/$FILE -o varlibs/obj_$NAME/${FILE%.cu}.o
OBJS=$(ls $CS/build/*.o | grep -v "/${FILE%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o varlibs/$NAME.so $OBJS varlibs/obj_$NAME/${FILE%.cu}.o -cudart static
echo varlibs/$NAME.so
