for L in default exp/lib_mx64.so exp/lib_mx128.so exp/lib_mx256.so exp/lib_lq16.so exp/lib_lq24.so; do
  if [ $L = default ]; then E=""; else E="TCCD_LIB=$L"; fi
  env $E python tools/gpu/lane_probe.py 1 1000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp4.log
  env $E python tools/gpu/lane_probe.py 3 50000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp4.log
done
