mkdir -p gpurun_out
(while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem27.log; sleep 1; done) &
MP=$!
JET_HIER_STATS=1 JET_COARSEN_TIMES=1 timeout 900 python scripts/probe_rmat_big.py 27 fast > gpurun_out/rmat_27.log 2>&1
echo "rc=$? max mem MiB: $(sort -n gpurun_out/mem27.log | tail -1)"
kill $MP
grep -v "^  L\|COARSEN n=" gpurun_out/rmat_27.log | tail -16
