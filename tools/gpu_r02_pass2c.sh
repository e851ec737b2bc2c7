for l in default acc64_kb2 acc64_2; do
  if [ $l = default ]; then LP=""; else LP="varlibs/$l.so"; fi
  echo "== $l accuracy S=64"; CNMF_LIB_PATH=$LP PA_S=64 timeout 200 python tools/pass_accuracy.py | grep -v "^  T"
  echo "== $l speed"; CNMF_LIB_PATH=$LP IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py 20000 100000 64 2>&1 | tail -2
done
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
