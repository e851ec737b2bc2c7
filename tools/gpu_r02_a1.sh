for l in a1kb1 a1kb1_32 a1kb2; do
  echo "== $l"; CNMF_LIB_PATH=varlibs/$l.so IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py 20000 100000 64 2>&1 | tail -2
  CNMF_LIB_PATH=varlibs/$l.so IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py 20000 100000 32 2>&1 | tail -2
  CNMF_LIB_PATH=varlibs/$l.so PA_S=64 timeout 200 python tools/pass_accuracy.py | grep -v "^  T" | tail -2
  CNMF_LIB_PATH=varlibs/$l.so timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -s -k "config4 or config1" 2>&1 | grep -E "projector|passed|failed"
done
