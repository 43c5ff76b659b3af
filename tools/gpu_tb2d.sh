for lib in tbnp tbp2 tbp4; do
  B200FD_LIB=build/$lib/libb200fd.so timeout 200 python tools/time_orders.py --orders 4,8 --variants tb2 --nt 20 --tag $lib
done > gpurun_out/tb2d.log 2>&1
B200FD_LIB=build/tbp2/libb200fd.so timeout 300 python -m pytest tests/test_gpu_acoustic.py -q -p no:cacheprovider -k tb2 -x >> gpurun_out/tb2d.log 2>&1
B200FD_LIB=build/tbp4/libb200fd.so timeout 300 python -m pytest tests/test_gpu_acoustic.py -q -p no:cacheprovider -k tb2 -x >> gpurun_out/tb2d.log 2>&1
cat gpurun_out/tb2d.log
