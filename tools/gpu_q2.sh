# queue2 (two y rows per thread) vs queue: parity, then per-order timing.
set -x
python -m pytest tests/test_gpu_acoustic.py -q -x -k "queue2" -p no:cacheprovider > gpurun_out/q2_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/q2_tests.log
python tools/time_orders.py --orders 2,4,6,8,12,16 --nt 40 --variants queue,queue2 > gpurun_out/q2_orders.jsonl 2>&1; echo "orders rc=$?"
cat gpurun_out/q2_orders.jsonl
