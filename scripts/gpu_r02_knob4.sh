echo "fixed salt: $(timeout 900 python scripts/quality_knob.py 2>&1 | tail -1)"
echo "vary salt:  $(JET_MATCH_VARY_SALT=1 timeout 900 python scripts/quality_knob.py 2>&1 | tail -1)"
