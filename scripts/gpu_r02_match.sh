mkdir -p gpurun_out
JET_K=64 JET_MATCH_STATS=1 timeout 300 python scripts/probe_rmat_big.py 22 fast > gpurun_out/rmat22_match.log 2>&1
grep FAST gpurun_out/rmat22_match.log | awk '{print $2, $3, $4, $5}' | head -150
