for l in base kb4 ast3 ast2 nacc1; do
  echo "== $l"; CNMF_LIB_PATH=varlibs/$l.so IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py 20000 100000 64 2>&1 | tail -2
done
