mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" build/libjet_512_1.so build/libjet_256_3.so build/libjet_256_4.so build/libjet_384_2.so; do
  echo "== variant ${v:-default}"
  JET_LIB=$v timeout 300 python scripts/probe.py 128 64 2>&1 | grep -E "^rep 2|refine_level"
done
JET_PHASES=1 timeout 300 python scripts/probe.py 128 64 > gpurun_out/phases.log 2>&1
