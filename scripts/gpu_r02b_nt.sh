# Non-temporal staging stores: e2e split vs the previous build; GPU tests that upload host graphs
mkdir -p gpurun_out
for i in 1 2 3; do for v in cur build/libjet_base3.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "$v $(JET_SPIN=1 timeout 300 python scripts/e2e_times.py 2>&1 | tail -1)"
done; done
unset JET_LIB
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
