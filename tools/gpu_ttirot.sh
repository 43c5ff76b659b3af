timeout 300 python tools/time_tti.py 30 > gpurun_out/ttirot.log 2>&1
B200FD_LIB=build/ttirot/libb200fd.so timeout 300 python tools/time_tti.py 30 >> gpurun_out/ttirot.log 2>&1
B200FD_LIB=build/ttirot/libb200fd.so timeout 600 python -m pytest tests/test_tti.py -q -p no:cacheprovider -x -m gpu >> gpurun_out/ttirot.log 2>&1
cat gpurun_out/ttirot.log
