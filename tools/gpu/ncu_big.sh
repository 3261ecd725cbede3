mkdir -p gpurun_out
timeout 300 python tools/profile_one.py --order random --n 268435456 --warmup 1 > gpurun_out/pbig.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5a.csv python tools/profile_one.py --order random --n 268435456 --warmup 1 > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_finish_warp|k_scatter_keys|k_count" -s 3 -c 3 -o gpurun_out/big_full python tools/profile_one.py --order random --n 268435456 --warmup 1 > gpurun_out/ncu_f.log 2>&1
