mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_finish_warp" -s 4 -c 1 -o gpurun_out/fin_full python tools/profile_one.py --order random --n 268435456 --warmup 0 > gpurun_out/ncu_fin.log 2>&1
