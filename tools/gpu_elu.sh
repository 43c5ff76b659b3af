timeout 300 python tools/time_elastic.py 30 > gpurun_out/elu.log 2>&1
B200FD_LIB=build/elu9/libb200fd.so timeout 300 python tools/time_elastic.py 30 >> gpurun_out/elu.log 2>&1
B200FD_LIB=build/elu9/libb200fd.so timeout 600 python -m pytest tests/test_elastic.py -q -p no:cacheprovider -x -m gpu >> gpurun_out/elu.log 2>&1
cat gpurun_out/elu.log
