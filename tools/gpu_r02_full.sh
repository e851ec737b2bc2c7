timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
timeout 900 python bench.py > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
timeout 600 python bench.py --config 1 > gpurun_out/bench1.log 2>&1; echo "rc=$?" >> gpurun_out/bench1.log
