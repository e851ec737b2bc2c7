for l in r64_96_112 r48_104_112 r56_104_104; do
  echo "== $l"; CNMF_LIB_PATH=varlibs/$l.so IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py 20000 100000 64 2>&1 | tail -2
done
