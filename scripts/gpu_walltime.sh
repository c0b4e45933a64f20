# median wall time of the device-resident partition (throughput mode) per library, alternating
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in default $EXTRA_LIBS; do
    if [ $v = default ]; then unset JET_LIB; else export JET_LIB=$v; fi
    echo "$v $(timeout 300 python scripts/walltime.py 2>&1 | tail -1)"
  done
done
