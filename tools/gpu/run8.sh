for L in exp/lib_m3u.so exp/lib_m4.so exp/lib_m2u.so; do
  TCCD_LIB=$L python tools/gpu/lane_probe.py 3 50000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp8.log
done
