set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b=$?
timeout 600 python bench.py --workload c5a --steps 10 --no-cpu-baseline > gpurun_out/bench_c5a.json 2> gpurun_out/bench_c5a.err
for w in c5b c5c c3 c4 c1; do timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_*.json
