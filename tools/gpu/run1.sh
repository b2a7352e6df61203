set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_lane.py -x -q > gpurun_out/t_lane.log 2>&1; echo "lane rc=$?" >> gpurun_out/t_lane.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/b3.json 2> gpurun_out/b3.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_lane.py > gpurun_out/t_all.log 2>&1; echo "all rc=$?" >> gpurun_out/t_all.log
