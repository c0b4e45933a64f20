# Budgeted (out-of-memory) hierarchy: parity test, then R-MAT 2^26 / 2^27 k=1024 probes.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_hierarchy_budget.py -m gpu -x -q > gpurun_out/pytest_budget.log 2>&1; tail -3 gpurun_out/pytest_budget.log
(while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem.log; sleep 1; done) &
MP=$!
for s in ${SCALES:-26 27}; do
  JET_HIER_STATS=1 JET_COARSEN_TIMES=1 timeout ${TMO:-900} python scripts/probe_rmat_big.py $s ${MODES:-fast,det} > gpurun_out/rmat_$s.log 2>&1
  echo "== scale $s rc=$?" >> gpurun_out/rmat_$s.log; echo "max mem MiB: $(sort -n gpurun_out/mem.log | tail -1)" >> gpurun_out/rmat_$s.log
  grep -v "^  L\|COARSEN n=" gpurun_out/rmat_$s.log | tail -12
done
kill $MP
