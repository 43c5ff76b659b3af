timeout 1500 python -m pytest tests/test_tti.py tests/test_elastic.py tests/test_gpu_full_length.py tests/test_host.py -q -p no:cacheprovider -m gpu -k "float64 or config4 or config5" > gpurun_out/f64_tests.log 2>&1; echo "rc=$?"
FDR_PARITY_REPORT=gpurun_out/parity_report45.json timeout 900 python -m pytest tests/test_gpu_full_length.py -q -p no:cacheprovider -k "config4 or config5" >> gpurun_out/f64_tests.log 2>&1
tail -15 gpurun_out/f64_tests.log; cat gpurun_out/parity_report45.json
