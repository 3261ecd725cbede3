mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scatter_keys|k_count" -s 0 -c 2 -o gpurun_out/scat_full python tools/profile_one.py --order random --n 268435456 --warmup 0 > gpurun_out/ncu_s.log 2>&1
