# Per-iteration refinement trace of the headline (throughput mode)
mkdir -p gpurun_out
JET_TRACE=1 JET_MODE=fast timeout 300 python scripts/one_partition.py 128 64 1 > gpurun_out/trace_fast.log 2>&1; echo rc=$?
grep -c TRACE gpurun_out/trace_fast.log
