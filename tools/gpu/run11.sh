python tools/gpu/lane_probe.py 3 50000000 > gpurun_out/lp11.log 2>&1
python tools/gpu/lane_probe.py 1 1000000 >> gpurun_out/lp11.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lane.py -x -q >> gpurun_out/lp11.log 2>&1; echo "tests rc=$?" >> gpurun_out/lp11.log
