# Full ncu capture of the cluster kernel on config 1 (one 100-step launch),
# 1 and 4 clusters.
for c in 1 4; do
  B200FD_CLUSTERS=$c python tools/small_probe.py 64x64x64 cluster 100 > gpurun_out/pc$c.log 2>&1 && \
  B200FD_CLUSTERS=$c ncu --set full --clock-control none --import-source on -k regex:acoustic_cluster -s 2 -c 1 \
      -o gpurun_out/cl$c python tools/small_probe.py 64x64x64 cluster 100 > gpurun_out/ncu_cl$c.log 2>&1
done
ls gpurun_out
