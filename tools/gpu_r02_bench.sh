timeout 900 python bench.py > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
timeout 600 python bench.py --config 1 > gpurun_out/bench1.log 2>&1; echo "rc=$?" >> gpurun_out/bench1.log
