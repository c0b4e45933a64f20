timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; tail -2 gpurun_out/pytest_gpu2.log
VARIANTS="base: nocl:JET_LV_CLUSTER_N=0 cl4k:JET_LV_CLUSTER_N=4096 cl16k:JET_LV_CLUSTER_N=16384 cl256k:JET_LV_CLUSTER_N=262144 b512_1:JET_LIB=build/libjet_512_1.so b256_3:JET_LIB=build/libjet_256_3.so" bash scripts/gpu_ab_env.sh
JET_PHASES=1 JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/probe_cl.log 2>&1
JET_LV_CLUSTER_N=0 JET_PHASES=1 JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/probe_nocl.log 2>&1
grep -E "^rep|  L" gpurun_out/probe_cl.log; grep -E "^rep|  L" gpurun_out/probe_nocl.log
