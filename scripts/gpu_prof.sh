mkdir -p gpurun_out
timeout 300 python scripts/profile_sweeps.py > gpurun_out/prof_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name regex:k_agg --launch-count 10 -o gpurun_out/sweeps -f python scripts/profile_sweeps.py > gpurun_out/ncu_sweeps.log 2>&1
tail -3 gpurun_out/ncu_sweeps.log; ls -la gpurun_out
