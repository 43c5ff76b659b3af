for lib in default qf1 qf2 default qf2; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  timeout 300 python tools/time_orders.py --orders 2,8,16 --variants queue --nt 40 --tag $lib
done > gpurun_out/qfperf.log 2>&1
cat gpurun_out/qfperf.log
