mkdir -p gpurun_out
SR_RES_DEBUG=1 timeout 300 python tools/profile_one.py --order random > gpurun_out/dbg.log 2>&1
SR_RES_DEBUG=1 timeout 300 python tools/profile_one.py --order few_unique >> gpurun_out/dbg.log 2>&1
SR_RES_DEBUG=1 timeout 300 python tools/profile_one.py --order random --n 300000 >> gpurun_out/dbg.log 2>&1
