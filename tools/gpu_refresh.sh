# Round-end evidence for the headline kernel: bench line, launch list, full ncu capture.
set -x
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-sweep --no-e2e --no-cpu --no-configs --no-fp64"
$B > gpurun_out/b1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_o8.csv $B > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:acoustic_queue -s 750 -c 1 -o gpurun_out/full_o8 $B > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
