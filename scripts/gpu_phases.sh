mkdir -p gpurun_out
JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases.log 2>&1
JET_TRACE=1 timeout 300 python scripts/one_partition.py 128 64 1 > gpurun_out/trace.log 2>&1
