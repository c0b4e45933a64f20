mkdir -p gpurun_out
(while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem.log; sleep 2; done) &
MP=$!
for s in ${SCALES:-25 26 27}; do
  timeout ${TMO:-600} python scripts/probe_rmat_big.py $s fast,det > gpurun_out/rmat_$s.log 2>&1
  echo "== scale $s rc=$?"; grep -v "^  L" gpurun_out/rmat_$s.log | tail -8
  echo "max mem MiB: $(sort -n gpurun_out/mem.log | tail -1)"
done
kill $MP
