timeout 900 python -m pytest tests/test_tti.py tests/test_elastic.py -q -p no:cacheprovider -m gpu -k "float64" > gpurun_out/f64b.log 2>&1; echo "rc=$?"
grep -E "assert .* < |passed|failed" gpurun_out/f64b.log | head
FDR_PARITY_REPORT=gpurun_out/parity_report45.json timeout 900 python -m pytest tests/test_gpu_full_length.py -q -p no:cacheprovider -k "config4 or config5" >> gpurun_out/f64b.log 2>&1
tail -2 gpurun_out/f64b.log; cat gpurun_out/parity_report45.json
