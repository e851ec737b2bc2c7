timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
timeout 900 python bench.py > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
CNMF_ADMM_PROFILE=1 ITERS=500 timeout 300 python tools/admm_timing.py > gpurun_out/admm_spec_prof.log 2>&1
