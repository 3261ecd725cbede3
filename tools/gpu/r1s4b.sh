# ncu evidence for C1 (resident, 1M) and C5c (multi-kernel int64 128M), then their bench lines citing the captures
mkdir -p gpurun_out/r1s4b /tmp/ncu
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s4b/launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o /tmp/ncu/full_c1 python tools/profile_one.py --order random --n 1000000 > /tmp/ncu/ncu_full_c1.log 2>&1
python tools/make_profile_summary.py r1s4_c1 gpurun_out/r1s4b/launches_c1.csv /tmp/ncu/full_c1.ncu-rep c1 > gpurun_out/r1s4b/summ_c1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s4b/launches_c5c.csv python bench.py --workload c5c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c5c.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"^(k_scatter_keys|k_count|k_finish_warp|k_presort_scan)$" -c 8 -o /tmp/ncu/full_c5c python tools/profile_one.py --order random --n 134217728 --dtype int64 --warmup 0 > /tmp/ncu/ncu_full_c5c.log 2>&1
python tools/make_profile_summary.py r1s4_c5c gpurun_out/r1s4b/launches_c5c.csv /tmp/ncu/full_c5c.ncu-rep c5c > gpurun_out/r1s4b/summ_c5c.log 2>&1
tail -3 /tmp/ncu/ncu_full_c5c.log > gpurun_out/r1s4b/ncu_full_c5c_tail.log
cp profiles/r1s4_c1_* profiles/r1s4_c5c_* gpurun_out/r1s4b/ 2>/dev/null
timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/r1s4b/bench_c1.json 2> gpurun_out/r1s4b/bench_c1.err
timeout 600 python bench.py --workload c5c --no-cpu-baseline > gpurun_out/r1s4b/bench_c5c.json 2> gpurun_out/r1s4b/bench_c5c.err
du -sh gpurun_out
