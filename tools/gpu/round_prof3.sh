# round-end evidence (small outputs only): tests, benches, launch lists; ncu --set full
# captures are summarised on the box (tools/make_profile_summary.py) and the reports dropped
mkdir -p gpurun_out/rp2
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/rp2/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rp2/gpu_tests.log
timeout 600 python bench.py > gpurun_out/rp2/bench_c2.json 2> gpurun_out/rp2/bench_c2.err
for w in c1 c3 c4 c5a c5b c5c c2d c2l16; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/rp2/bench_$w.json 2> gpurun_out/rp2/bench_$w.err; done
timeout 300 python bench.py --impl reference --steps 3 > gpurun_out/rp2/ref_c2.json 2> gpurun_out/rp2/ref_c2.err
mkdir -p /tmp/ncu
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rp2/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o /tmp/ncu/full_c2 python tools/profile_one.py --order random > /tmp/ncu/ncu_full_c2.log 2>&1
python tools/make_profile_summary.py r1s3f_c2 gpurun_out/rp2/launches_c2.csv /tmp/ncu/full_c2.ncu-rep c2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rp2/launches_c5a.csv python bench.py --workload c5a --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c5a.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"^(k_scatter_keys|k_count|k_finish_warp|k_presort_scan)$" -c 8 -o /tmp/ncu/full_c5a python tools/profile_one.py --order random --n 268435456 --warmup 0 > /tmp/ncu/ncu_full_c5a.log 2>&1
python tools/make_profile_summary.py r1s3f_c5a gpurun_out/rp2/launches_c5a.csv /tmp/ncu/full_c5a.ncu-rep c5a > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rp2/launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"^(k_scatter|k_count|k_finish)$" -s 6 -c 3 -o /tmp/ncu/full_c4 python tools/timeline_pairs.py > /tmp/ncu/ncu_full_c4.log 2>&1
python tools/make_profile_summary.py r1s3f_c4 gpurun_out/rp2/launches_c4.csv /tmp/ncu/full_c4.ncu-rep c4 > /dev/null 2>&1
cp profiles/r1s3f_* gpurun_out/rp2/ 2>/dev/null
du -sh gpurun_out
