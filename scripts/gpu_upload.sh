# e2e upload time vs host staging threads (throughput mode, headline workload)
mkdir -p gpurun_out; nproc
for th in 8 16 32 64; do
  echo "== threads $th"
  JET_UPLOAD_THREADS=$th JET_MODE=fast timeout 300 python scripts/one_partition.py 128 64 3 2>&1 | grep -E "e2e partition" | tail -2
done
