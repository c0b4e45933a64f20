for i in 1 2; do
for v in cur ${VARIANTS}; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "$v grid128: $(timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
done
done
for v in cur ${VARIANTS}; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "$v rmat22: $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
  echo "$v rgg24: $(timeout 300 python scripts/ab_time.py rgg 24 256 3 2>&1 | tail -1)"
done
