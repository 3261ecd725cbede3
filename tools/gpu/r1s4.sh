# round-end evidence for the current commit: ncu first (so the bench lines cite this capture), then tests, smoke, benches
mkdir -p gpurun_out/r1s4 /tmp/ncu
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s4/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o /tmp/ncu/full_c2 python tools/profile_one.py --order random > /tmp/ncu/ncu_full_c2.log 2>&1
python tools/make_profile_summary.py r1s4_c2 gpurun_out/r1s4/launches_c2.csv /tmp/ncu/full_c2.ncu-rep c2 > gpurun_out/r1s4/summ.log 2>&1
cp profiles/r1s4_c2_* gpurun_out/r1s4/ 2>/dev/null
tail -5 /tmp/ncu/ncu_full_c2.log > gpurun_out/r1s4/ncu_full_tail.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r1s4/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r1s4/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s4/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1s4/smoke.log
timeout 600 python bench.py > gpurun_out/r1s4/bench_c2.json 2> gpurun_out/r1s4/bench_c2.err
for w in c1 c3 c4 c5a c5b c5c c2d c2l16; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r1s4/bench_$w.json 2> gpurun_out/r1s4/bench_$w.err; done
timeout 300 python bench.py --impl reference --steps 3 > gpurun_out/r1s4/ref_c2.json 2> gpurun_out/r1s4/ref_c2.err
du -sh gpurun_out
