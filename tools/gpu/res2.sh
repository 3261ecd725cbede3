mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/res_test.log 2>&1; echo "resident tests rc=$?" >> gpurun_out/res_test.log
SR_TIMING=1 timeout 300 python tools/latency.py 2000000 > gpurun_out/lat.log 2>&1
