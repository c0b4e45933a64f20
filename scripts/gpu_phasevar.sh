# JET_PHASES totals (throughput mode) for the in-tree library and EXTRA_LIBS
mkdir -p gpurun_out
for v in default $EXTRA_LIBS; do
  if [ $v = default ]; then unset JET_LIB; else export JET_LIB=$v; fi
  JET_PHASES=1 JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/pv.log 2>&1
  echo "== $v"; grep -E "^rep 2" gpurun_out/pv.log; python scripts/phase_totals.py gpurun_out/pv.log ${TOPN:-8}
done
