# Two-step kernel: parity tests, then timings against the single-step kernel.
timeout 600 python -m pytest tests/test_gpu_acoustic.py -q -p no:cacheprovider -k "tb2" -x > gpurun_out/tb2_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/tb2_tests.log
timeout 300 python tools/time_orders.py --orders 2,4,6,8 --variants queue,tb2 --nt 40 > gpurun_out/tb2_time.log 2>&1; echo "time rc=$?"
cat gpurun_out/tb2_time.log
