for shp in "20000 100000 64" "20000 100000 32" "10000 5000 32"; do
  echo "== $shp"; IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py $shp 2>&1 | tail -2
done
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
timeout 900 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench4.log 2>&1
