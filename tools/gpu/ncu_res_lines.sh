mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/profile_one.py --order random > /tmp/ncu/p1.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o /tmp/ncu/res python tools/profile_one.py --order random > /tmp/ncu/ncu1.log 2>&1
python tools/ncu_lines.py /tmp/ncu/res.ncu-rep k_resident 80 > gpurun_out/res_lines_stall.txt 2>&1
python tools/ncu_lines.py /tmp/ncu/res.ncu-rep k_resident 80 inst > gpurun_out/res_lines_inst.txt 2>&1
