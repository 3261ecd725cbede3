mkdir -p gpurun_out
timeout 120 python tools/profile_one.py --order random > gpurun_out/p1.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o gpurun_out/res_c2_random python tools/profile_one.py --order random > gpurun_out/ncu_res.log 2>&1
