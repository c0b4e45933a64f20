# grid_res + merged contraction readbacks vs the PB4 build: A/B (128^3, R-MAT 2^22), host waits, -m gpu suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
for v in cur build/libjet_pb4.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "grid $v $(timeout 300 python scripts/ab_time.py grid 128 64 9 2>&1 | tail -1)"
  echo "rmat $v $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
done; done
unset JET_LIB
JET_SYNC_STATS=1 JET_MODE=fast timeout 300 python scripts/one_partition.py 128 64 2 2>&1 | tail -4
JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/probe_cur.log 2>&1
head -22 gpurun_out/probe_cur.log | tail -21; tail -1 gpurun_out/probe_cur.log
