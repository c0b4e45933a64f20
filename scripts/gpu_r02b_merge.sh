# Row merge with the next row's header prefetched (75 regs) vs 64/51-register caps vs the previous build
mkdir -p gpurun_out
for i in 1 2; do
for v in cur build/libjet_mm4.so build/libjet_mm5.so build/libjet_base4.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "grid $v $(timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
  JET_MODE=fast timeout 300 python scripts/probe.py 128 64 2>&1 | grep -E 'contract_rows'
done; done
unset JET_LIB
echo "rmat cur $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
echo "rmat base4 $(JET_LIB=build/libjet_base4.so timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
