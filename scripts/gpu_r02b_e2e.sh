# e2e split (upload / device / download) vs host staging threads; old download path for comparison
mkdir -p gpurun_out; nproc; lscpu | grep -E 'Model name|Socket|NUMA node\(s\)|^CPU\(s\)'
for th in 16 32 64; do JET_SPIN=1 JET_UPLOAD_THREADS=$th timeout 300 python scripts/e2e_times.py 2>&1 | tail -1; done
JET_SPIN=1 JET_LIB=build/libjet_pb4.so timeout 300 python scripts/e2e_times.py 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -q -x -k "parity or edge or pipeline or host" > gpurun_out/pytest_sub.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_sub.log
