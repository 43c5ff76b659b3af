# Deferred-dyz A/B for tti_pack (config 4) plus the TTI parity / canary / full-length tests
timeout 900 python -m pytest tests/test_tti.py tests/test_gpu_canary.py -q -p no:cacheprovider -x -k "tti or TTI" > gpurun_out/ttidefer_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ttidefer_tests.log
timeout 900 python -m pytest tests/test_gpu_full_length.py -q -p no:cacheprovider -x -k "config4" > gpurun_out/ttidefer_full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/ttidefer_full.log
for rep in 1 2; do
  for v in default defer_noalt nodefer; do
    if [ $v = default ]; then unset B200FD_LIB; else export B200FD_LIB=$PWD/build/$v/libb200fd.so; fi
    echo "== $v rep $rep"; timeout 300 python tools/time_tti.py 30 2>&1 | head -1
  done
done
unset B200FD_LIB
