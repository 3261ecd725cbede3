# iteration check: GPU tests, C2 bench, latency breakdown
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; echo "all gpu rc=$?" >> gpurun_out/gpu_all.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python tools/latency.py 2000000 > gpurun_out/lat.log 2>&1
