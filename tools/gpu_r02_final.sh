# round-2 evidence: tests, bench lines for every configuration, launch lists, ncu captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
timeout 900 python bench.py > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
for c in 1 0 2 3; do timeout 900 python bench.py --config $c > gpurun_out/bench$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench$c.log; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
# launch lists of the bench commands (one warm-up + one timed step, no e2e / cpu legs)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l1.log 2>&1
# full captures: the pass kernel inside the configs[4] bench step, the NNLS refit of the XRAY job
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"stream_pass2" -s 24 -c 2 -o gpurun_out/prof4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_p4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nnls_kernel -s 44 -c 1 -o gpurun_out/nnls_prof python tools/xray_plain.py > gpurun_out/ncu_nnls.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"admm_spec" -c 1 -o gpurun_out/admm_spec_prof python bench.py --config 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_spec.log 2>&1
