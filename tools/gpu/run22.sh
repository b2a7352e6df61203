python bench.py --steps 20 --warmup 5 > gpurun_out/b22.json 2> gpurun_out/b22.err
python bench.py --config 1 --steps 20 --warmup 5 > gpurun_out/b22c1.json 2> gpurun_out/b22c1.err
python bench.py --config 0 --steps 20 --warmup 5 --no-e2e > gpurun_out/b22c0.json 2> gpurun_out/b22c0.err
python bench.py --config 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/b22c2.json 2> gpurun_out/b22c2.err
