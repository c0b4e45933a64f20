# Session start on a fresh build: -m gpu suite, smoke, per-level phase breakdown (128^3 throughput), short bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
JET_MODE=fast JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases.log 2>&1
python scripts/phase_totals.py gpurun_out/phases.log 40 > gpurun_out/phase_totals.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.log
