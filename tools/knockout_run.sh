# time forward/transpose passes per knockout library at a configs[4]-like slab
M=${M:-20000}; N=${N:-100000}
for S in 64 32; do
for l in base nomma nosplit noepi nosttm noepi_nosttm nomma_noepi; do
  echo "== $l S=$S"; CNMF_LIB_PATH=varlibs/$l.so IMPL=1 REPS=5 timeout 300 python tools/pass_bench.py $M $N $S 2>&1 | tail -2
done; done
