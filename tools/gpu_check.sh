# Parity suite, smoke and the default bench line on one GPU.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.log 2>&1
python -m pytest tests -q -m gpu -p no:cacheprovider --durations=25 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/gpu_tests.log
