# Cluster-synchronised level kernel on the tiniest levels only (JET_LV_CLUSTER_N)
mkdir -p gpurun_out
for i in 1 2; do for v in 0 2200 4000 8000; do
  echo "CLUSTER_N=$v grid $(JET_LV_CLUSTER_N=$v timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
done; done
for v in 0 2200 4000; do
  echo "CLUSTER_N=$v rmat $(JET_LV_CLUSTER_N=$v timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
  echo "CLUSTER_N=$v rgg $(JET_LV_CLUSTER_N=$v timeout 300 python scripts/ab_time.py rgg 24 256 3 2>&1 | tail -1)"
done
JET_LV_CLUSTER_N=4000 JET_MODE=fast JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases_cl.log 2>&1
grep -E "^PHASES L1[2-7]" gpurun_out/phases_cl.log | tail -12
exit 0
