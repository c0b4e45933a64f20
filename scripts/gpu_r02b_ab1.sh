# Propose row batching A/B (PB=4 in-tree vs PB=1/2 variants) on 128^3 and R-MAT 2^22,
# per-class device times, and ncu source captures of a small level kernel (L7) and L11.
mkdir -p gpurun_out
for i in 1 2; do
for v in cur build/libjet_pb1.so build/libjet_pb2.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "grid $v $(timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
  echo "rmat $v $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
done; done
unset JET_LIB
JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/probe_pb4.log 2>&1
JET_LIB=build/libjet_pb1.so JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/probe_pb1.log 2>&1
grep -E 'propose|accept' gpurun_out/probe_pb4.log gpurun_out/probe_pb1.log
SKIPS="10 6" bash scripts/gpu_r02_ncu_small.sh
