timeout 600 python -m pytest tests -m gpu -q --timeout 300 -k "residual_pass or relative_error or snmf" > gpurun_out/resid_tests.log 2>&1; echo "rc=$?" >> gpurun_out/resid_tests.log
timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
