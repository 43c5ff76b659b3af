# Queue kernel tile-height A/B (one-wave grids at 512^2: 8 x 37 tiles of 64 x 14).
for lib in default ty14 ty14n5; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  timeout 300 python tools/time_orders.py --orders 2,4,8,12,16 --variants queue --nt 40 --tag $lib
done > gpurun_out/ty.log 2>&1
cat gpurun_out/ty.log
