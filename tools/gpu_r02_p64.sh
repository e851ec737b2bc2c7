for shp in "20000 100000 64" "20000 100000 32"; do
  echo "== $shp"; IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py $shp 2>&1 | tail -2
done
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "pass or compress or subspace or range or config4" > gpurun_out/pass2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pass2_tests.log
