for q in 50000000 25000000 12500000 6250000; do
  python bench.py --queries $q --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print($q, round(d['ms_per_step'],2), '%.3g'%d['value'], {k: round(v['ms'],2) for k,v in d['roofline']['stages'].items()})" >> gpurun_out/scale_proxy.log
done
