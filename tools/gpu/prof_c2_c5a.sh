# Phase stamps of the resident kernel (C2 orders) and ncu --set full captures of
# the C2 resident kernel and the C5a pipeline kernels (real launches only).
set -x
mkdir -p gpurun_out
for o in random nearly few_unique reversed; do
  SR_TIMING=1 timeout 120 python tools/profile_one.py --order $o --warmup 3 > gpurun_out/st_$o.log 2>&1
done
timeout 300 python tools/profile_one.py --order random --warmup 2 > gpurun_out/plain_c2.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resident -s 2 -c 1 \
   -o gpurun_out/r2_c2_res -f python tools/profile_one.py --order random --warmup 2 > gpurun_out/ncu_c2.log 2>&1
timeout 300 python tools/profile_one.py --order random --n 268435456 --warmup 1 > gpurun_out/plain_c5a.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on \
   -k regex:'k_count|k_scatter_keys|k_finish_warp|k_presort_scan|k_finish<' -s 14 -c 14 \
   -o gpurun_out/r2_c5a -f python tools/profile_one.py --order random --n 268435456 --warmup 1 > gpurun_out/ncu_c5a.log 2>&1
echo done
