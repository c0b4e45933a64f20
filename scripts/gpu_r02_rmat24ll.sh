mkdir -p gpurun_out
JET_HIER_BUDGET_MB=4000 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rmat24_launches.csv python scripts/probe_rmat_big.py 24 fast > gpurun_out/rmat24_ll.log 2>&1; echo "rc=$?"
