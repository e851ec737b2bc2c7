set -x
L=paper_1505_04650_b200/libcnmf_b200.so
cp $L /tmp/ns8.so
for v in ns8 ns16; do
  if [ $v = ns16 ]; then cp tools/libcnmf_b200_ns16.so $L; else cp /tmp/ns8.so $L; fi
  echo "=== $v"
  timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "paired or repeated" 2>&1 | tail -3
  for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'])"; done
  timeout 300 python tools/compress_timing.py 20000 10000 20 2>&1 | head -2
done
cp /tmp/ns8.so $L
