mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name regex:k_agg_small --launch-count 4 -o gpurun_out/sweeps -f python scripts/profile_sweeps.py > gpurun_out/ncu_sweeps.log 2>&1
tail -2 gpurun_out/ncu_sweeps.log
