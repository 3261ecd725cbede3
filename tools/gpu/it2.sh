# iteration check: resident tests first, then all GPU tests, C2 bench, stamps
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/res_test.log 2>&1; echo "resident rc=$?" >> gpurun_out/res_test.log
for o in random few_unique; do SR_TIMING=1 timeout 60 python tools/profile_one.py --order $o --warmup 3 > gpurun_out/st_$o.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; echo "all gpu rc=$?" >> gpurun_out/gpu_all.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python tools/latency.py 2000000 > gpurun_out/lat.log 2>&1
