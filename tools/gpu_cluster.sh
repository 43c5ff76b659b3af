# Cluster-kernel parity + small-grid timings (config 1 and neighbours).
python -m pytest tests -q -m gpu -p no:cacheprovider -k "cluster or failure or canary or smoke or config1" > gpurun_out/cl_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/cl_tests.log
for c in 1 2 4 8; do B200FD_CLUSTERS=$c python tools/small_probe.py 64x64x64 cluster 100; done > gpurun_out/cl_probe.log 2>&1
python tools/small_probe.py 64x64x64,40x36x44,48x48x48 cluster,persistent,queue 100 >> gpurun_out/cl_probe.log 2>&1
cat gpurun_out/cl_probe.log
