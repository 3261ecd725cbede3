# ncu evidence for C3 (16M partial-order sweep) and C4 (stable pairs): launch lists + --set full of the dominant scatter
mkdir -p gpurun_out/r1s4c /tmp/ncu
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s4c/launches_c3.csv python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"^(k_scatter_keys|k_count|k_presort_scan)$" -c 3  # NOTE: caught only tiny level-2 launches; summary not kept -o /tmp/ncu/full_c3 python tools/profile_one.py --order swaps_1e3 --n 16777216 --warmup 0 > /tmp/ncu/ncu_full_c3.log 2>&1
python tools/make_profile_summary.py r1s4_c3 gpurun_out/r1s4c/launches_c3.csv /tmp/ncu/full_c3.ncu-rep c3 > gpurun_out/r1s4c/summ_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s4c/launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"^(k_scatter|k_count)$" -s 4 -c 2 -o /tmp/ncu/full_c4 python tools/timeline_pairs.py > /tmp/ncu/ncu_full_c4.log 2>&1
python tools/make_profile_summary.py r1s4_c4 gpurun_out/r1s4c/launches_c4.csv /tmp/ncu/full_c4.ncu-rep c4 > gpurun_out/r1s4c/summ_c4.log 2>&1
tail -3 /tmp/ncu/ncu_full_c3.log /tmp/ncu/ncu_full_c4.log > gpurun_out/r1s4c/ncu_tails.log
cp profiles/r1s4_c3_* profiles/r1s4_c4_* gpurun_out/r1s4c/ 2>/dev/null
timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r1s4c/bench_c3.json 2> gpurun_out/r1s4c/bench_c3.err
timeout 300 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/r1s4c/bench_c4.json 2> gpurun_out/r1s4c/bench_c4.err
