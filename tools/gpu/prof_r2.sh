# Round-2 evidence: resident phase stamps (C2 orders), ncu --set full of the C2
# resident kernel and of every kernel of one C5a (256M int32 random) sort
# (second sort of the process: -s 11 -c 11 skips the warm-up sort's 11 launches).
set -x
mkdir -p gpurun_out/prof
for o in random nearly few_unique reversed; do
  SR_TIMING=1 timeout 120 python tools/profile_one.py --order $o --warmup 3 > gpurun_out/prof/st_$o.log 2>&1
done
timeout 300 python tools/profile_one.py --order random --warmup 2 > gpurun_out/prof/plain_c2.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resident -s 2 -c 1 \
   -o gpurun_out/prof/c2_res -f python tools/profile_one.py --order random --warmup 2 > gpurun_out/prof/ncu_c2.log 2>&1
timeout 300 python tools/profile_one.py --order random --n 268435456 --warmup 1 > gpurun_out/prof/plain_c5a.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_count|k_scatter_keys|k_finish|k_presort_scan' -s 11 -c 11 \
   -o gpurun_out/prof/c5a -f python tools/profile_one.py --order random --n 268435456 --warmup 1 > gpurun_out/prof/ncu_c5a.log 2>&1
echo done
