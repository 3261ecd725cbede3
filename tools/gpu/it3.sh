# quick sanity (short timeouts), then resident tests, stamps, bench
mkdir -p gpurun_out
SR_TIMING=1 timeout 30 python tools/profile_one.py --order random --warmup 1 > gpurun_out/st_random.log 2>&1; echo "rc=$?" >> gpurun_out/st_random.log
timeout 300 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/res_test.log 2>&1; echo "resident rc=$?" >> gpurun_out/res_test.log
for o in random few_unique nearly; do SR_TIMING=1 timeout 30 python tools/profile_one.py --order $o --warmup 3 > gpurun_out/st_$o.log 2>&1; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
