# Ordered tail: payload loads issued beside the key loads (rank path); parity suite, A/B, phase totals
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for i in 1 2 3; do for v in cur build/libjet_base8.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "grid $v $(timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
  [ $i = 1 ] && echo "rmat $v $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
done; done
unset JET_LIB
for v in cur build/libjet_base8.so; do
  if [ $v != cur ]; then export JET_LIB=$v; fi
  JET_MODE=fast JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases_tail.log 2>&1
  echo "$v"; python scripts/phase_totals.py gpurun_out/phases_tail.log 40 | grep -E 'rb_tail|total'
done
exit 0
