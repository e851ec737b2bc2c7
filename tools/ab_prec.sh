for L in main lotrunc; do
  if [ $L = main ]; then unset CNMF_LIB_PATH; else export CNMF_LIB_PATH=$PWD/oldlib/$L.so; fi
  echo "=== $L"; python tools/subspace_precision.py 2>&1 | tail -1
  IMPL=1 python tools/pass_bench.py 40000 50000 64; IMPL=1 python tools/pass_bench.py 40000 50000 32
done
