# Per-phase/per-level breakdown of the level kernels (128^3 k=64 throughput) + ncu of coarse levels.
mkdir -p gpurun_out
JET_MODE=fast JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases.log 2>&1
python scripts/phase_totals.py gpurun_out/phases.log 40 > gpurun_out/phase_totals.txt 2>&1
grep "^  L" gpurun_out/phases.log | tail -20
cat gpurun_out/phase_totals.txt | head -45
for sk in ${SKIPS:-6 11}; do
JET_MODE=fast timeout 900 ncu --set full --clock-control none --import-source on --kernel-name "regex:k_level($|<)" \
  --launch-skip $sk --launch-count 1 -o gpurun_out/k_level_skip$sk -f python scripts/one_partition.py 128 64 1 > gpurun_out/ncu_skip$sk.log 2>&1
echo "ncu skip $sk rc=$?"
done
