# Two-step kernel A/B: wait and fence variants (timing only for tbw0).
for lib in default tbw1 tbw0 tbf0; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  timeout 200 python tools/time_orders.py --orders 4,8 --variants tb2 --nt 20 --tag $lib
done > gpurun_out/tb2b.log 2>&1
unset B200FD_LIB
cat gpurun_out/tb2b.log
