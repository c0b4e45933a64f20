# Sticky hub proposals (throughput matching): R-MAT time/cut vs the previous build, quality gates, sharding parity
mkdir -p gpurun_out
for i in 1 2; do for v in cur build/libjet_base5.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "rmat $v $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
done; done
unset JET_LIB
timeout 600 python scripts/quality_knob.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_throughput_mode.py tests/test_sharding.py -m gpu -q 2>&1 | tail -4
