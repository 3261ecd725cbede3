mkdir -p gpurun_out
SR_TIMING=1 timeout 300 python tools/latency.py 2000000 > gpurun_out/lat.log 2>&1
timeout 300 python tools/timeline.py 2000000 random > gpurun_out/tl_random.log 2>&1
timeout 300 python tools/timeline.py 2000000 few_unique > gpurun_out/tl_few.log 2>&1
timeout 300 python tools/launch_overhead.py > gpurun_out/lo.log 2>&1
