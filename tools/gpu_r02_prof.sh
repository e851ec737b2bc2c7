# launch list of the configs[4] bench command (one warm-up + one timed step, no e2e/cpu legs)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l1.log 2>&1
# full captures at configs[4] size: the pass kernel, the row sweep, the core step
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"stream_pass2|row_sweep|core_step" -s 20 -c 3 -o gpurun_out/prof4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_p4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stream_pass2" -s 4 -c 1 -o gpurun_out/prof1 python bench.py --config 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_p1.log 2>&1
