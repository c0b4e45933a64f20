mkdir -p gpurun_out
for sk in ${SKIPS:-6 11}; do
JET_MODE=fast timeout 900 ncu --set full --clock-control none --import-source on --kernel-name "regex:k_level($|<)" \
  --launch-skip $sk --launch-count 1 -o gpurun_out/k_level_skip$sk -f python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_skip$sk.log 2>&1
echo "ncu skip $sk rc=$?"
done
