mkdir -p gpurun_out
SR_TIMING=1 timeout 300 python tools/latency.py 2000000 > gpurun_out/lat.log 2>&1
for o in random reversed nearly few_unique; do SR_TIMING=1 timeout 60 python tools/profile_one.py --order $o --warmup 3 > gpurun_out/st_$o.log 2>&1; done
timeout 300 python tools/launch_overhead.py > gpurun_out/lo.log 2>&1
