timeout 900 python -m pytest tests -m gpu -x -q -k "admm or distributed or shard" > gpurun_out/admm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/admm_tests.log
timeout 300 python tools/admm_stream_profile.py > gpurun_out/admm_prof2.log 2>&1
