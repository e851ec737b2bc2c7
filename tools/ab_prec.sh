for L in main kb1 kb4 acc64 kb1acc64 libcnmf_b200; do
  if [ $L = main ]; then unset CNMF_LIB_PATH; else export CNMF_LIB_PATH=$PWD/oldlib/$L.so; fi
  echo "=== $L"; python tools/subspace_precision.py 2>&1 | tail -1
done
unset CNMF_LIB_PATH
export IMPL=1
for L in main kb1 acc64; do
  if [ $L = main ]; then unset CNMF_LIB_PATH; else export CNMF_LIB_PATH=$PWD/oldlib/$L.so; fi
  echo "=== perf $L"; python tools/pass_bench.py 40000 50000 64; python tools/pass_bench.py 40000 50000 32
done
