# bench headline (device ms, e2e ms, deterministic ms) for the in-tree library and EXTRA_LIBS, alternating
mkdir -p gpurun_out
for i in 1 2; do
  for v in default $EXTRA_LIBS; do
    if [ $v = default ]; then unset JET_LIB; else export JET_LIB=$v; fi
    JET_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --no-extra-configs --no-cpu-baseline > gpurun_out/lb.log 2>&1
    echo "$v $(tail -1 gpurun_out/lb.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), round(d["e2e"]["partition_time_s"]*1e3,1), round(d["deterministic_mode"]["ms_per_step"],1))' 2>&1 | tail -1)"
  done
done
