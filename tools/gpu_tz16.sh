for lib in default tz16; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  echo "== $lib"; timeout 300 python tools/time_tti.py 30 2>&1 | head -2
done > gpurun_out/tz16.log 2>&1
B200FD_LIB=build/tz16/libb200fd.so timeout 900 python -m pytest tests/test_tti.py -q -p no:cacheprovider -m gpu -x >> gpurun_out/tz16.log 2>&1
cat gpurun_out/tz16.log | tail -8
