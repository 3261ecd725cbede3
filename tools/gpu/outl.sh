mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_outlier.py -x -q > gpurun_out/outl_test.log 2>&1; echo "rc=$?" >> gpurun_out/outl_test.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --workload c3 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c5b --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
