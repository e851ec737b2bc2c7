for l in default acc64_kb2 acc64_2; do
  if [ $l = default ]; then LP=""; else LP="varlibs/$l.so"; fi
  echo "== $l"; CNMF_LIB_PATH=$LP timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -s -k "config4 or config1" 2>&1 | grep -E "projector|passed|failed"
  echo "== $l V1"; CNMF_PASS_V=1 CNMF_LIB_PATH=$LP timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -s -k "config4" 2>&1 | grep -E "projector|passed|failed"
done
