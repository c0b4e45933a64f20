# diagnostics run on the GPU box: smoke, per-level phase clocks, ncu of the L0 level kernel
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name "regex:k_level($|<)" --launch-skip 14 --launch-count 1 -o gpurun_out/k_level_L0 -f python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_full.log 2>&1
