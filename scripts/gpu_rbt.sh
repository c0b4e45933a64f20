# per-call rb_tail section cycles (needs the RBT printf build) for the default lib and EXTRA_LIBS
mkdir -p gpurun_out
for v in default $EXTRA_LIBS; do
  if [ $v = default ]; then unset JET_LIB; else export JET_LIB=$v; fi
  JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/rbt_$(basename $v).log 2>&1
  echo "== $v"; grep -E "^rep 2|refine_level" gpurun_out/rbt_$(basename $v).log
  python scripts/rbt_summary.py gpurun_out/rbt_$(basename $v).log
done
