set -x
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
timeout 600 python bench.py --config 1 > gpurun_out/bench1.log 2>&1; echo "rc=$?" >> gpurun_out/bench1.log
