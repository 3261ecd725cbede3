# A/B: resident launch through the cached graph node vs direct cooperative launch
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/res_test.log 2>&1; echo "resident rc=$?" >> gpurun_out/res_test.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_graph$i.json 2> gpurun_out/bench_graph$i.err
SR_NO_GRAPH=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_direct$i.json 2> gpurun_out/bench_direct$i.err
done
timeout 300 python bench.py --workload c1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1g.json 2>&1
SR_NO_GRAPH=1 timeout 300 python bench.py --workload c1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1d.json 2>&1
