for lib in default u9 ubr1 default; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  timeout 300 python tools/time_orders.py --orders 8 --variants queue --nt 60 --tag $lib
done > gpurun_out/u9.log 2>&1
cat gpurun_out/u9.log
