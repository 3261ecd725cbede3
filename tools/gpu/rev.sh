mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q > gpurun_out/res_test.log 2>&1; echo "rc=$?" >> gpurun_out/res_test.log
SR_TIMING=1 timeout 30 python tools/profile_one.py --order reversed --warmup 3 > gpurun_out/st_reversed.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_rev.json 2> gpurun_out/bench_rev.err
