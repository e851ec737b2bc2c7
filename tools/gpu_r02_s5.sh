timeout 600 python -m pytest tests -m gpu -x -q -k "admm_stream or rank_above or shard" > gpurun_out/admm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/admm_tests.log
timeout 300 python tools/admm_iter_timing.py 2>&1 | grep -v -i warn > gpurun_out/admm_iter.log
timeout 300 python tools/admm_stream_profile.py 2>&1 | grep -v -i warn | head -8 > gpurun_out/admm_prof.log
