# Host staging threads for the e2e upload (16-core box): repeated medians
mkdir -p gpurun_out; nproc
for i in 1 2 3; do for th in 16 24 32 48; do JET_SPIN=1 JET_UPLOAD_THREADS=$th timeout 300 python scripts/e2e_times.py 2>&1 | tail -1; done; done
