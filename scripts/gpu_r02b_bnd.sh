# Boundary-only Jetlp sweeps only above JET_BND_MIN_N vertices (smaller levels sweep every row, no collect phase)
mkdir -p gpurun_out
for i in 1 2; do for v in 0 30000 100000 300000; do
  echo "BND_MIN_N=$v grid $(JET_BND_MIN_N=$v timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
  [ $i = 1 ] && echo "BND_MIN_N=$v rmat $(JET_BND_MIN_N=$v timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
  [ $i = 1 ] && echo "BND_MIN_N=$v rgg $(JET_BND_MIN_N=$v timeout 300 python scripts/ab_time.py rgg 24 256 3 2>&1 | tail -1)"
done; done
JET_BND_MIN_N=100000 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_bnd.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_bnd.log
exit 0
