mkdir -p gpurun_out
for cfg in "0 3 0" "4 3 0" "4 3 1024" "4 3 2048" "4 2 1024" "3 3 1024"; do
  set -- $cfg
  echo "CP=$1 FROM=$2 P=$3: $(python - <<PY 2>&1 | tail -1
import os, runpy, sys
PY
JET_CPV=$1 JET_CPF=$2 JET_CP_P=$3 timeout 900 python -c "
import sys; sys.argv=['q']
import paper_2304_13194_b200.config as C, os
C.RefinerConfig.coarse_patience = int(os.environ['JET_CPV']); C.RefinerConfig.coarse_patience_from = int(os.environ['JET_CPF'])
exec(open('scripts/quality_knob.py').read())
" 2>&1 | tail -1)"
done
