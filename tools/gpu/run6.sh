timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_all6.log 2>&1; echo "all rc=$?" >> gpurun_out/t_all6.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke6.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke6.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b3_6.json 2> gpurun_out/b3_6.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref6.json 2> gpurun_out/ref6.err
