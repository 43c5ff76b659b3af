# Round-end evidence: GPU parity suite (with the fp64 error report), smoke,
# bench line, launch list, FLOP/DRAM counters and full ncu captures of the
# production kernels (each ncu pass only after the same command exited 0
# without ncu).
set -x
FDR_PARITY_REPORT=gpurun_out/parity_report.json python -m pytest tests -q -rs -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -12 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-sweep --no-e2e --no-cpu --no-configs --no-fp64"
$B > gpurun_out/b1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_o8.csv $B > gpurun_out/ncu1.log 2>&1
bash tools/ncu_flops.sh
ncu --set full --clock-control none --import-source on -k regex:acoustic_queue -s 750 -c 1 -o gpurun_out/full_o8 $B > gpurun_out/ncu2.log 2>&1
python tools/time_tti.py 6 > gpurun_out/tti6.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tti_pack -s 4 -c 1 -o gpurun_out/full_tti python tools/time_tti.py 6 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
# summaries on the box (the reports exceed what comes back comfortably)
(python tools/ncu_summary.py gpurun_out/full_o8.ncu-rep; python tools/ncu_src_stalls.py gpurun_out/full_o8.ncu-rep) > gpurun_out/r02_ncu_full_bench_o8.txt 2>&1
(python tools/ncu_summary.py gpurun_out/full_tti.ncu-rep; python tools/ncu_src_stalls.py gpurun_out/full_tti.ncu-rep) > gpurun_out/r02_ncu_full_tti_pack_config4.txt 2>&1
