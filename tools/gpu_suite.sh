# Full GPU parity suite + smoke.
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
