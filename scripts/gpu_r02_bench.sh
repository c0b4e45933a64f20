# Bench (default args) + reference arm + launch list of the headline
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ("value","ms_per_step","cutsize","gpu_launches")}, d["roofline"]["frac"], d["e2e"]["value"], [ (c["workload"][:22], round(c["partition_time_s"],3), c["cutsize"], c.get("cut_ratio_vs_cpu_ref"), c.get("cut_ratio_vs_deterministic")) for c in d["configs_measured"]], d["deterministic_mode"]["ms_per_step"])'
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.log
JET_MODE=fast timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/one_partition.py 128 64 1 > gpurun_out/launches.log 2>&1; echo "ncu rc=$?"
