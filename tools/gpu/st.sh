mkdir -p gpurun_out
for o in random few_unique; do SR_TIMING=1 timeout 30 python tools/profile_one.py --order $o --warmup 3 > gpurun_out/st_$o.log 2>&1; done
