timeout 900 python -m pytest tests/test_tti.py tests/test_gpu_dense_receivers.py tests/test_gpu_canary.py -q -p no:cacheprovider -x > gpurun_out/tti_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tti_tests.log
timeout 300 python tools/time_tti.py 30 > gpurun_out/tti_time.log 2>&1; cat gpurun_out/tti_time.log
