mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_scatter$" -s 3 -c 1 -o gpurun_out/pairs_full python tools/timeline_pairs.py > gpurun_out/ncu_p.log 2>&1
