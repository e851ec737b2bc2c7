for shp in "10000 5000 32" "4000 3000 32" "20000 100000 32"; do
  echo "== $shp"; IMPL=1 REPS=20 timeout 300 python tools/pass_bench.py $shp 2>&1 | tail -2
done
timeout 600 python bench.py --config 1 --no-e2e --no-cpu-baseline > gpurun_out/bench1.log 2>&1
