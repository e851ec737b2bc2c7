for v in 2; do
  for shp in "20000 100000 64" "20000 100000 32" "10000 5000 32"; do
    echo "== V$v $shp"; CNMF_PASS_V=$v IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py $shp 2>&1 | tail -2
  done
done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "pass or compress or subspace or range" > gpurun_out/pass2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pass2_tests.log
