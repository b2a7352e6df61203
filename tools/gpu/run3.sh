python tools/gpu/lane_probe.py 3 4000000 > gpurun_out/lp3.log 2>&1
python tools/gpu/lane_probe.py 3 50000000 >> gpurun_out/lp3.log 2>&1
python tools/gpu/lane_probe.py 1 1000000 >> gpurun_out/lp3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all3.log 2>&1; echo "all rc=$?" >> gpurun_out/t_all3.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b3_3.json 2> gpurun_out/b3_3.err
