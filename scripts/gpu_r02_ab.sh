# Parity subset + A/B of device time (128^3 k=64 and R-MAT 2^22) between the in-tree library and variants.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_big.py tests/test_hierarchy_budget.py tests/test_throughput_mode.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; tail -3 gpurun_out/pytest_ab.log
for i in 1 2; do
for v in cur ${VARIANTS:-build/libjet_base.so}; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "$v grid128: $(timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
done
done
for v in cur ${VARIANTS:-build/libjet_base.so}; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "$v rmat22: $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
done
unset JET_LIB
JET_MODE=fast JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases.log 2>&1
python scripts/phase_totals.py gpurun_out/phases.log 40 > gpurun_out/phase_totals.txt 2>&1
grep "^  L" gpurun_out/phases.log | tail -18
head -30 gpurun_out/phase_totals.txt
