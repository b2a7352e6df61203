for L in default exp/lib_tail128.so exp/lib_tailoff.so; do
for q in 50000000 6250000; do
  if [ $L = default ]; then E=""; else E="TCCD_LIB=$L"; fi
  env $E python bench.py --queries $q --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print('$L', $q, round(d['ms_per_step'],2), '%.3g'%d['value'], {k: round(v['ms'],2) for k,v in d['roofline']['stages'].items()})" >> gpurun_out/tail.log
done; done
python tools/gpu/lane_probe.py 3 6250000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/tail.log
