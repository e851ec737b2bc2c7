for shp in "20000 100000 64" "20000 100000 32" "10000 5000 32"; do
  echo "== $shp"; IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py $shp 2>&1 | tail -2
done
timeout 900 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench4.log 2>&1
REPS=1 IMPL=1 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:stream_pass2 -c 2 python tools/pass_bench.py 20000 100000 64 > gpurun_out/ncu_l2.log 2>&1
