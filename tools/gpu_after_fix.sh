timeout 600 python tools/small_stress.py 20 > gpurun_out/after_fix.log 2>&1
timeout 600 python tools/tb2_stress.py 2 6 >> gpurun_out/after_fix.log 2>&1
timeout 600 python tools/tb2_stress.py 8 4 >> gpurun_out/after_fix.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider >> gpurun_out/after_fix.log 2>&1; echo "tests rc=$?" >> gpurun_out/after_fix.log
grep -v "^rep" gpurun_out/after_fix.log | tail -12
