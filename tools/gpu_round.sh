set -x
python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-sweep --no-e2e --no-cpu --no-configs"
$B > gpurun_out/b1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_o8.csv $B > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:acoustic_queue -s 750 -c 1 -o gpurun_out/full_o8 $B > gpurun_out/ncu2.log 2>&1
python tools/time_tti.py 6 > gpurun_out/tti.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tti_stream -s 4 -c 1 -o gpurun_out/full_tti python tools/time_tti.py 6 > gpurun_out/ncu3.log 2>&1
python tools/time_elastic.py 6 > gpurun_out/el.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:el_stream -s 8 -c 2 -o gpurun_out/full_el python tools/time_elastic.py 6 > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out
