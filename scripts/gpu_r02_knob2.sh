for ct in 200 1000 2000 4000 8000; do
  echo "CT=$ct: $(CT=$ct timeout 900 python scripts/quality_knob.py 2>&1 | tail -1)"
done
