for v in 0 1000 3000 8000; do
  echo "SKIP=$v: $(JET_SKIP_LEVEL_N=$v timeout 900 python scripts/quality_knob.py 2>&1 | tail -1)"
done
