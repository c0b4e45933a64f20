mkdir -p gpurun_out
JET_MODE=fast timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name "regex:k_level<.bool.1>" --launch-count 1 -o gpurun_out/r02_k_level_L0_fast -f python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_full1.log 2>&1; echo "full L0 rc=$?"
JET_K=64 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name "regex:k_level<.bool.1>" --launch-count 1 -o gpurun_out/r02_k_level_L0_rmat22 -f python scripts/probe_rmat_big.py 22 fast > gpurun_out/ncu_full2.log 2>&1; echo "full rmat L0 rc=$?"
ls -la gpurun_out/*.ncu-rep
