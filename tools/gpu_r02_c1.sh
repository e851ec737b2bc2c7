for l in acc2_64 kb1_32; do
  echo "== $l"; for i in 1 2 3; do CNMF_LIB_PATH=varlibs/$l.so timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -s -k "config1" 2>&1 | grep -E "projector"; done
  CNMF_LIB_PATH=varlibs/$l.so IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py 10000 5000 32 2>&1 | tail -2
  CNMF_LIB_PATH=varlibs/$l.so IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py 20000 100000 32 2>&1 | tail -2
done
echo "== V1"; for i in 1 2 3; do CNMF_PASS_V=1 timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -s -k "config1" 2>&1 | grep -E "projector"; done
