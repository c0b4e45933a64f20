# Round-2 GPU check: full -m gpu suite, then compute-sanitizer (memcheck,
# racecheck, synccheck) over the kernel-parity tests (small graphs).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
SAN="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in memcheck racecheck synccheck; do
  timeout 900 $SAN --tool $tool python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
    -k "match or contract or select or afterburner or jetlp or rebalance or jet_refine or cutsize" \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
