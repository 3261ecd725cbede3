# Round-2 evidence for the current commit: GPU suite (normal and checked
# library), smoke, every workload's bench line, the reference arm, the C2 and
# C5a launch lists, ncu --set full of the C2 resident kernel (random) and of
# the C5a pipeline kernels (real launches: the second sort of the process),
# summarised here into profiles/TAG_* (see the end).  usage: bash tools/gpu/evidence_r2.sh TAG
set -x
TAG=${1:-r2s7}
O=gpurun_out/ev
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu_full.log 2>&1
SR_CHECKED_LIB=1 timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu_checked.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in c1 c3 c4 c5b c5c c2d c2l16 c2l256; do
  timeout 600 python bench.py --workload $w --sub none --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 300 python bench.py --l2 flush --sub none --no-cpu-baseline > $O/bench_c2_flush.json 2> $O/bench_c2_flush.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference_c2.json 2> $O/reference_c2.err
# launch lists (cold-cache, serialised: shares, not absolutes); the second C2 list without ncu's
# cache control: the DRAM reads per launch show that the rotating inputs come from HBM
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/c2_launches.csv python bench.py --steps 20 --warmup 3 --sub none --no-cpu-baseline --no-e2e > $O/ncu_c2_list.log 2>&1
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/c2_nocc_launches.csv python bench.py --steps 20 --warmup 3 --sub none --no-cpu-baseline --no-e2e > $O/ncu_c2_nocc_list.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/c5a_launches.csv python tools/profile_one.py --order random --n 268435456 --warmup 1 > $O/ncu_c5a_list.log 2>&1
# --set full captures
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resident -s 3 -c 1 \
  -o $O/c2_res -f python tools/profile_one.py --order random --warmup 3 --flush > $O/ncu_c2_full.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:'k_count|k_scatter_keys|k_finish_warp|k_presort_scan|k_finish<' -s 14 -c 16 \
  -o $O/c5a_full -f python tools/profile_one.py --order random --n 268435456 --warmup 1 > $O/ncu_c5a_full.log 2>&1
python tools/ncu_lines.py $O/c2_res.ncu-rep k_resident 40 > $O/c2_res_lines.txt 2>&1
ls -la $O
echo done
# then, here: python tools/make_profile_summary.py TAG_c2 gpurun_out/ev/c2_launches.csv gpurun_out/ev/c2_res.ncu-rep c2
#             python tools/make_profile_summary.py TAG_c5a gpurun_out/ev/c5a_launches.csv gpurun_out/ev/c5a_full.ncu-rep c5a
