# Throughput matching: proposers that found no free neighbour skip their row in later rounds (exact)
mkdir -p gpurun_out
for i in 1 2 3; do for v in cur build/libjet_base6.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "grid $v $(timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
  echo "rmat $v $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
  JET_MODE=fast timeout 300 python scripts/probe.py 128 64 2>&1 | grep -E '^propose'
done; done
unset JET_LIB
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
