mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/res_test.log 2>&1; echo "resident tests rc=$?" >> gpurun_out/res_test.log
SR_TIMING=1 timeout 300 python tools/latency.py 2000000 > gpurun_out/lat.log 2>&1
timeout 300 python tools/profile_one.py --order random > gpurun_out/p1.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 2 -c 1 -o gpurun_out/res_random python tools/profile_one.py --order random > gpurun_out/ncu1.log 2>&1
