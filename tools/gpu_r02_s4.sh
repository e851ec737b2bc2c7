# round-2 re-entry check: GPU tests, every configuration's bench line
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
for c in 4 1 0 2 3; do
  timeout 900 python bench.py --config $c > gpurun_out/bench$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench$c.log
done
