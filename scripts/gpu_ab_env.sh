# A/B: each VARIANT is "name:ENV=VAL,ENV2=VAL2" (":" alone = base); two rounds, alternating
mkdir -p gpurun_out
for r in 1 2; do
for v in $VARIANTS; do
  name=${v%%:*}; envs=$(echo ${v#*:} | tr ',' ' ')
  echo "$name $(env $envs timeout 300 python scripts/ab_time.py ${WL:-grid 128 64} 2>&1 | tail -1)"
done
done
