for L in exp/lib_k96.so exp/lib_k128.so exp/lib_k256.so; do
  TCCD_LIB=$L python tools/gpu/lane_probe.py 3 50000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp9.log
  TCCD_LIB=$L python tools/gpu/lane_probe.py 1 1000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp9.log
done
