# Shared-memory pressure of the acoustic queue kernel per order (round 2):
# smoke, per-order timing, then ncu L1/shared-memory counters at orders 8 and 16.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python tools/time_orders.py --orders 2,4,8,12,16 --nt 40 > gpurun_out/orders.jsonl 2>&1; echo "orders rc=$?"
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_reads.sum,l1tex__data_bank_writes.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__memory_throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second
for o in 8 16; do
  python tools/prof_step.py --order $o --nt 6 --random > gpurun_out/p$o.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:acoustic_queue -s 3 -c 1 --csv python tools/prof_step.py --order $o --nt 6 --random > gpurun_out/smem_o$o.csv 2>&1
done
ncu --query-metrics --chip gb100 2>/dev/null | grep -i -E "l1tex__data_bank|lsu_wavefronts|l1tex__m_|smem|shared" > gpurun_out/metric_names.txt
ls -la gpurun_out
