mkdir -p gpurun_out
SR_HOSTPROF=1 timeout 60 python tools/profile_one.py --order reversed --warmup 5 > gpurun_out/hp_graph.log 2>&1
SR_NO_GRAPH=1 SR_HOSTPROF=1 timeout 60 python tools/profile_one.py --order reversed --warmup 5 > gpurun_out/hp_direct.log 2>&1
SR_HOSTPROF=1 timeout 60 python tools/profile_one.py --order random --warmup 5 > gpurun_out/hp_random.log 2>&1
timeout 120 python tools/pyoverhead.py > gpurun_out/pyover.log 2>&1
