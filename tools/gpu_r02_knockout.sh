bash tools/knockout_run.sh > gpurun_out/knockout.log 2>&1
REPS=1 IMPL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_pass -c 1 -o gpurun_out/pass64 python tools/pass_bench.py 20000 100000 64 > gpurun_out/ncu64.log 2>&1
