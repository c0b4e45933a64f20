mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_throughput_mode.py tests/test_gpu_parity.py tests/test_configs.py tests/test_reference_big.py tests/test_hierarchy_budget.py tests/test_sharding.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; tail -3 gpurun_out/pytest_ab.log
for v in cur ${VARIANTS:-build/libjet_base.so}; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "$v grid128: $(timeout 300 python scripts/ab_time.py grid 128 64 5 2>&1 | tail -1)"
  echo "$v rmat22: $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
  echo "$v rgg24: $(timeout 300 python scripts/ab_time.py rgg 24 256 3 2>&1 | tail -1)"
done
unset JET_LIB
JET_K=64 JET_COARSEN_TIMES=1 timeout 300 python scripts/probe_rmat_big.py 22 fast > gpurun_out/rmat22_c.log 2>&1
grep -v "^  L" gpurun_out/rmat22_c.log | tail -25
