# level-kernel totals (throughput mode) under environment variants: ENVS="A=1 B=2,C=3" (comma = same run)
mkdir -p gpurun_out
for e in base $ENVS; do
  if [ $e = base ]; then envs=""; else envs=$(echo $e | tr ',' ' '); fi
  env $envs JET_PHASES=1 JET_MODE=fast timeout 300 python scripts/probe.py 128 64 > gpurun_out/ev.log 2>&1
  echo "== $e $(grep -E '^rep 2' gpurun_out/ev.log | cut -c1-60) $(python scripts/phase_totals.py gpurun_out/ev.log 1 | tail -1)"
done
