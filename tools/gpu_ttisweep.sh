for lib in default ttins3 ttins5 ttity8; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  echo "== $lib"; timeout 300 python tools/time_tti.py 30 2>&1 | head -1
done > gpurun_out/ttisweep.log 2>&1
cat gpurun_out/ttisweep.log
