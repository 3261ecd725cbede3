mkdir -p gpurun_out
timeout 300 python tools/profile_one.py --order ${1:-random} > gpurun_out/p1.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o gpurun_out/res_${1:-random} python tools/profile_one.py --order ${1:-random} > gpurun_out/ncu1.log 2>&1
