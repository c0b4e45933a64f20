# Two-hop frontier threshold (deterministic mode): A/B of the mesh levels on the frontier kernel
mkdir -p gpurun_out
for v in 16384 0 1024; do
  echo "TH_FRONTIER_MIN=$v grid $(JET_TH_FRONTIER_MIN=$v timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
  JET_TH_FRONTIER_MIN=$v JET_MODE=det timeout 300 python scripts/probe.py 128 64 2>&1 | grep -E 'two_hop|th_'
done
JET_TH_FRONTIER_MIN=0 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_th0.log 2>&1; echo "pytest th0 rc=$?"; tail -1 gpurun_out/pytest_th0.log
