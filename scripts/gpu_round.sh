# Round evidence on the GPU box: tests, smoke, bench (both arms), ncu launch list + full capture
# of the finest-level refinement kernel (throughput mode: the bench headline; 18 levels).
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1
JET_MODE=fast timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/one_partition.py 128 64 1 > gpurun_out/launches.log 2>&1
JET_MODE=fast timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name "regex:k_level($|<)" --launch-skip 17 --launch-count 1 -o gpurun_out/k_level_L0 -f python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_full.log 2>&1
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/launches.log gpurun_out/ncu_full.log; do echo "== $f"; tail -n 3 $f; done
