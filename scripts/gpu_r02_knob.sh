mkdir -p gpurun_out
for cfg in "4 3" "4 2" "4 1" "6 1" "3 3"; do
  set -- $cfg
  echo "CP=$1 FROM=$2: $(CPV=$1 CPF=$2 timeout 900 python scripts/quality_knob.py 2>&1 | tail -1)"
done
