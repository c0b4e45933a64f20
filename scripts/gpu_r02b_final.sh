# Round-2 (session b) evidence from the final build: -m gpu suite, smoke, bench (both arms), launch lists
# (throughput + deterministic headline, R-MAT 2^22), ncu --set full of the
# finest-level kernel (headline, R-MAT 2^22).
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
JET_MODE=fast timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_fast.csv python scripts/one_partition.py 128 64 1 > /dev/null 2>&1
JET_MODE=det timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_det.csv python scripts/one_partition.py 128 64 1 > /dev/null 2>&1
JET_K=64 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_rmat22.csv python scripts/probe_rmat_big.py 22 fast > /dev/null 2>&1
JET_MODE=fast timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name "regex:k_level<.bool.1>" --launch-count 1 -o gpurun_out/r02b_k_level_L0_fast -f python scripts/one_partition.py 128 64 1 > /dev/null 2>&1
JET_K=64 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name "regex:k_level<.bool.1>" --launch-count 1 -o gpurun_out/r02b_k_level_L0_rmat22 -f python scripts/probe_rmat_big.py 22 fast > /dev/null 2>&1
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log; do echo "== $f"; tail -n 3 $f; done
