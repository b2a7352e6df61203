for L in exp/lib_lq8.so exp/lib_lq12.so exp/lib_lq16.so exp/lib_lq16k32.so exp/lib_lq16k48.so exp/lib_lq16a2k.so; do
  TCCD_LIB=$L python tools/gpu/lane_probe.py 1 1000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp5.log
  TCCD_LIB=$L python tools/gpu/lane_probe.py 3 50000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp5.log
done
