# median event time of the headline partition under environment variants: ENVS="A=1 B=2,C=3"
mkdir -p gpurun_out
for i in 1 2; do
  for e in base $ENVS; do
    if [ $e = base ]; then envs=""; else envs=$(echo $e | tr ',' ' '); fi
    echo "$e $(env $envs timeout 300 python scripts/walltime.py 2>&1 | tail -1)"
  done
done
