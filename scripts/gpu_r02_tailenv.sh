for v in 2048 512 128 32 0; do
  echo "TAIL_GRID_MIN=$v: $(JET_TAIL_GRID_MIN=$v timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
done
