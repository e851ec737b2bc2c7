echo "== accuracy V1"; CNMF_PASS_V=1 timeout 200 python tools/pass_accuracy.py
echo "== accuracy V2 acc2"; CNMF_PASS_V=2 timeout 200 python tools/pass_accuracy.py
echo "== accuracy V2 acc1"; CNMF_LIB_PATH=varlibs/acc1.so CNMF_PASS_V=2 timeout 200 python tools/pass_accuracy.py
for shp in "20000 100000 64" "20000 100000 32" "10000 5000 32"; do
  echo "== V2 acc2 $shp"; CNMF_PASS_V=2 IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py $shp 2>&1 | tail -2
done
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "pass or compress or subspace or range" > gpurun_out/pass2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pass2_tests.log
