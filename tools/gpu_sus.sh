for lib in default sus200 sus2000; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  echo "== $lib"; timeout 300 python tools/time_tti.py 30 2>&1 | head -1
  timeout 300 python tools/time_elastic.py 20 2>&1 | head -1
  timeout 300 python tools/time_orders.py --orders 8 --variants queue --nt 40 --tag $lib
done > gpurun_out/sus.log 2>&1
cat gpurun_out/sus.log
