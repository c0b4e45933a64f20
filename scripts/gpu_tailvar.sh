mkdir -p gpurun_out
for g in 2048 0 256 512; do
  echo "== JET_TAIL_GRID_MIN=$g"
  JET_TAIL_GRID_MIN=$g JET_PHASES=1 JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/tv_$g.log 2>&1
  grep -E "^rep 2|refine_level" gpurun_out/tv_$g.log
  grep PHASES gpurun_out/tv_$g.log | grep strong | tail -17 | grep -oE "PHASES L[0-9]+|rb_tail=[0-9.]+|tail_sort=[0-9.]+" | paste - - - | tr '\n' ' '; echo
done
