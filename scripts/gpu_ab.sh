# A/B of the bench headline between the in-tree library and $BASE_LIB (alternating runs)
mkdir -p gpurun_out
for i in 1 2; do
  for v in cur $BASE_LIB; do
    if [ $v = cur ]; then unset JET_LIB; else export JET_LIB=$v; fi
    JET_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-extra-configs > gpurun_out/ab.log 2>&1
    echo "$v $(tail -1 gpurun_out/ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), d["cutsize"], round(d["e2e"]["partition_time_s"]*1e3,2), round(d["deterministic_mode"]["ms_per_step"],2))' 2>&1 | tail -1)"
  done
done
