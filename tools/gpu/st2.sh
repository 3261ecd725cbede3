mkdir -p gpurun_out
for o in random nearly; do SR_TIMING=1 timeout 60 python tools/profile_one.py --order $o --warmup 3 > gpurun_out/st_$o.log 2>&1; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
