mkdir -p gpurun_out
JET_K=64 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rmat22_launches.csv python scripts/probe_rmat_big.py 22 fast > gpurun_out/rmat22_launches.log 2>&1
echo "ncu rc=$?"
JET_K=64 JET_PHASES=1 timeout 300 python scripts/probe_rmat_big.py 22 fast x > gpurun_out/rmat22_phases.log 2>&1
python scripts/phase_totals.py gpurun_out/rmat22_phases.log 30 > gpurun_out/rmat22_phase_totals.txt 2>&1
cat gpurun_out/rmat22_phase_totals.txt
