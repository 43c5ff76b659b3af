for lib in default elcs default elcs; do
  if [ $lib = default ]; then unset B200FD_LIB; else export B200FD_LIB=build/$lib/libb200fd.so; fi
  echo "== $lib"; timeout 300 python tools/time_elastic.py 30 2>&1 | head -1
done > gpurun_out/elcs.log 2>&1
B200FD_LIB=build/elcs/libb200fd.so timeout 900 python -m pytest tests/test_elastic.py tests/test_gpu_canary.py -q -p no:cacheprovider -m gpu -x -k "elastic" >> gpurun_out/elcs.log 2>&1
timeout 900 python -m pytest tests/test_elastic.py -q -p no:cacheprovider -m gpu -x >> gpurun_out/elcs.log 2>&1
cat gpurun_out/elcs.log | tail -12
