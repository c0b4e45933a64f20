# Round-2 evidence pass: -m gpu suite, smoke, bench (our arm + reference arm),
# R-MAT scale 25/26/27 probes (configs[4] shape) with peak memory, ncu launch list.
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
(while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem.log; sleep 2; done) &
MP=$!
for s in ${SCALES:-26 27}; do
  timeout ${TMO:-600} python scripts/probe_rmat_big.py $s fast,det > gpurun_out/rmat_$s.log 2>&1
  echo "== scale $s rc=$?" >> gpurun_out/rmat_$s.log; echo "max mem MiB: $(sort -n gpurun_out/mem.log | tail -1)" >> gpurun_out/rmat_$s.log
done
kill $MP
JET_MODE=fast timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/one_partition.py 128 64 1 > gpurun_out/launches.log 2>&1
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/rmat_*.log gpurun_out/launches.log; do echo "== $f"; tail -n 4 $f; done
