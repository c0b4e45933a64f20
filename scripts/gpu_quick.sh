mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases.log 2>&1
grep -E "^rep 2|refine_level|match_resolve|total device" gpurun_out/phases.log
JET_PHASES=1 JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/probe_fast.log 2>&1
grep -E "^rep|refine_level|propose|accept|leaf|total device|  L" gpurun_out/probe_fast.log
for v in $EXTRA_LIBS; do echo "== $v"; JET_LIB=$v timeout 300 python scripts/probe.py 128 64 2>&1 | grep -E "^rep 2|refine_level"; done
JET_TRACE=1 JET_MODE=fast timeout 300 python scripts/one_partition.py 128 64 1 > gpurun_out/trace_fast.log 2>&1
