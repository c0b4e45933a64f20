# Level-kernel block shapes (threads, min blocks/SM): in-tree 512x2 vs 512x1 (no spills), 384x2, 256x3
mkdir -p gpurun_out
for i in 1 2; do
for v in cur build/libjet_512_1.so build/libjet_384_2.so build/libjet_256_3.so; do
  if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
  echo "grid $v $(timeout 300 python scripts/ab_time.py grid 128 64 7 2>&1 | tail -1)"
  [ $i = 1 ] && echo "rmat $v $(timeout 300 python scripts/ab_time.py rmat 22 64 3 2>&1 | tail -1)"
done; done
