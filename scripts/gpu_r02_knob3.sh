for cfg in "4 1" "4 0" "6 0" "8 0"; do
  set -- $cfg
  echo "CP=$1 FROM=$2: $(CPV=$1 CPF=$2 timeout 900 python scripts/quality_knob.py 2>&1 | tail -1)"
done
