# A/B: TMEM drain load width of the pass epilogue (8 / 16 / 32 columns per tcgen05.ld).
# The variant libraries are built first, here (no GPU needed), e.g. for 32:
#   nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
#        -DCNMF_PASS2_LDW=32 -c paper_1505_04650_b200/csrc/tc_pass2.cu -o /tmp/tc_pass2_32.o
#   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o varlibs/ldw32.so \
#        $(ls paper_1505_04650_b200/csrc/build/*.o | grep -v tc_pass2.o) /tmp/tc_pass2_32.o -cudart static
# (-DCNMF_VARIANT_NOMMA the same way gives the MMA knockout library of DESIGN.md)
for v in ldw8 default ldw32; do
  if [ $v = default ]; then unset CNMF_LIB_PATH; else export CNMF_LIB_PATH=$PWD/varlibs/$v.so; fi
  echo "== $v"
  IMPL=1 REPS=20 timeout 300 python tools/pass_bench.py 20000 100000 64 2>&1 | grep -v -i warn | tail -2
  IMPL=1 REPS=20 timeout 300 python tools/pass_bench.py 20000 100000 32 2>&1 | grep -v -i warn | tail -2
done
unset CNMF_LIB_PATH
timeout 900 python -m pytest tests -m gpu -x -q -k "pass or bit_reproducible or compress" 2>&1 | tail -3
CNMF_LIB_PATH=$PWD/varlibs/ldw32.so timeout 900 python -m pytest tests -m gpu -x -q -k "pass or bit_reproducible or compress" 2>&1 | tail -3
