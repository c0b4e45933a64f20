# Full -m gpu suite + smoke + A/B timings vs $VARIANTS
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for v in cur ${VARIANTS:-}; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "$v grid128: $(timeout 300 python scripts/ab_time.py grid 128 64 5 2>&1 | tail -1)"
  echo "$v rmat22: $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
  echo "$v rgg24: $(timeout 300 python scripts/ab_time.py rgg 24 256 3 2>&1 | tail -1)"
done
