mkdir -p gpurun_out/rp3 /tmp/ncu
timeout 600 python bench.py > gpurun_out/rp3/bench_c2.json 2> gpurun_out/rp3/bench_c2.err
timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/rp3/bench_c1.json 2> gpurun_out/rp3/bench_c1.err
timeout 300 python bench.py --workload c5c --no-cpu-baseline > gpurun_out/rp3/bench_c5c.json 2> gpurun_out/rp3/bench_c5c.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rp3/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o /tmp/ncu/full_c2 python tools/profile_one.py --order random > /tmp/ncu/ncu_full_c2.log 2>&1
python tools/make_profile_summary.py r1s3f_c2 gpurun_out/rp3/launches_c2.csv /tmp/ncu/full_c2.ncu-rep c2 > /dev/null 2>&1
cp profiles/r1s3f_c2_* gpurun_out/rp3/
