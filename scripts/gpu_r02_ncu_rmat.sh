# ncu source-level capture of one dense R-MAT 2^22 level kernel (k_level launches run coarsest first)
mkdir -p gpurun_out
JET_K=64 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name "regex:k_level($|<)" \
  --launch-skip ${SKIP:-12} --launch-count 1 -o gpurun_out/k_level_rmat22_skip${SKIP:-12} -f python scripts/probe_rmat_big.py 22 fast > gpurun_out/ncu_rmat.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_rmat.log
