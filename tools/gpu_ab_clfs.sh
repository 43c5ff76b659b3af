export B200FD_WAIT_CYCLES=$((1<<27))
B200FD_LIB=build/clfs/libb200fd.so timeout 900 python -m pytest tests/test_gpu_acoustic.py tests/test_gpu_canary.py tests/test_gpu_failure.py -q -m gpu -p no:cacheprovider -k "cluster or config1 or canary or failure" > gpurun_out/clfs_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/clfs_tests.log
O=gpurun_out/ab_clfs.jsonl; : > $O
for rep in 1 2 3; do
  timeout 200 python tools/small_probe.py 64x64x64,40x36x44 cluster 100 >> $O
  B200FD_LIB=build/clfs/libb200fd.so timeout 200 python tools/small_probe.py 64x64x64,40x36x44 cluster 100 | sed 's/"variant": "cluster"/"variant": "cluster+fastsync"/' >> $O
done
cat $O
