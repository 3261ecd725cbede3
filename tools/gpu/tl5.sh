mkdir -p gpurun_out
timeout 300 python tools/timeline.py 268435456 random > gpurun_out/tl_c5a.log 2>&1
timeout 300 python tools/timeline.py 134217728 random i64 > gpurun_out/tl_c5c.log 2>&1
timeout 300 python tools/timeline.py 16777216 runs1024 > gpurun_out/tl_c3r.log 2>&1
