set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/one_partition.py 128 64 1 > gpurun_out/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:k_level --launch-skip 14 --launch-count 1 -o gpurun_out/k_level_L0 python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/*.log
