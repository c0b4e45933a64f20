# Round-2 profile evidence (current build): launch lists (128^3 throughput +
# deterministic, R-MAT 2^22), full ncu captures of the finest-level kernel.
mkdir -p gpurun_out
JET_MODE=fast timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_fast.csv python scripts/one_partition.py 128 64 1 > /dev/null 2>&1; echo "ll fast rc=$?"
JET_MODE=det timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_det.csv python scripts/one_partition.py 128 64 1 > /dev/null 2>&1; echo "ll det rc=$?"
JET_K=64 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_rmat22.csv python scripts/probe_rmat_big.py 22 fast > /dev/null 2>&1; echo "ll rmat rc=$?"
JET_MODE=fast timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name "regex:k_level<1>" --launch-count 1 -o gpurun_out/r02_k_level_L0_fast -f python scripts/one_partition.py 128 64 1 > /dev/null 2>&1; echo "full L0 rc=$?"
JET_K=64 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name "regex:k_level<1>" --launch-count 1 -o gpurun_out/r02_k_level_L0_rmat22 -f python scripts/probe_rmat_big.py 22 fast > /dev/null 2>&1; echo "full rmat L0 rc=$?"
