# ncu source captures of the deterministic matching kernels on the finest level (128^3)
mkdir -p gpurun_out
JET_MATCH_STATS=1 JET_MODE=det timeout 300 python scripts/one_partition.py 128 64 1 2>&1 | grep -E 'FRONTIER|TWOHOP|TH' | head -20
JET_MODE=det timeout 900 ncu --set full --clock-control none --import-source on --kernel-name k_resolve_frontier \
  --launch-count 1 -o gpurun_out/k_resolve_L0 -f python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_resolve.log 2>&1; echo "ncu rc=$?"
JET_MODE=det timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_two_hop \
  --launch-count 1 -o gpurun_out/k_two_hop_L0 -f python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_twohop.log 2>&1; echo "ncu rc=$?"
