timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all2.log 2>&1; echo "all rc=$?" >> gpurun_out/t_all2.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/b3_2.json 2> gpurun_out/b3_2.err
timeout 300 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu > gpurun_out/b1_2.json 2> gpurun_out/b1_2.err
