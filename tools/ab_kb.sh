export IMPL=1
for L in main ast3 acc1 ast3kb8; do
  if [ $L = main ]; then unset CNMF_LIB_PATH; else export CNMF_LIB_PATH=$PWD/oldlib/$L.so; fi
  echo "=== $L"
  python tools/pass_bench.py 40000 50000 64
  python tools/pass_bench.py 20000 100000 64
done
