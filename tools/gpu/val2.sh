mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; echo "all gpu rc=$?" >> gpurun_out/gpu_all.log
timeout 600 python bench.py --workload c5a --no-cpu-baseline > gpurun_out/bench_c5a.json 2> gpurun_out/bench_c5a.err
bash tools/gpu/ncu_big.sh
