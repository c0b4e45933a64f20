# Weak rebalancing passes before strong (throughput mode): time and cut ratios, gate tests
mkdir -p gpurun_out
for wp in ${WPS:-3 4}; do
  echo "== WEAK_PASSES=$wp"
  JET_WEAK_PASSES=$wp timeout 600 python scripts/quality_knob.py 2>&1 | tail -3
  JET_WEAK_PASSES=$wp timeout 900 python -m pytest tests/test_throughput_mode.py -m gpu -q 2>&1 | tail -3
done
