# Bench line of the final build (our arm; both modes, all configs)
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err; echo "bench rc=$?"
tail -c 400 gpurun_out/bench_final.log
