mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; echo "all gpu rc=$?" >> gpurun_out/gpu_all.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --workload c3 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
