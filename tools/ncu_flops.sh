# ncu-counted FP32 work and DRAM bytes per launch of the TTI and elastic
# production kernels on their BASELINE configs (a few steps each).  FLOPs =
# FADD + FMUL + 2 FFMA + 2 FADD2 + 2 FMUL2 + 4 FFMA2 thread instructions.
M=smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
python tools/time_tti.py 6 > gpurun_out/tti_plain.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:tti_pack -s 4 -c 2 --csv python tools/time_tti.py 6 > gpurun_out/ncu_flops_tti.csv 2>&1
python tools/time_elastic.py 6 > gpurun_out/el_plain.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:el_ -s 8 -c 4 --csv python tools/time_elastic.py 6 > gpurun_out/ncu_flops_el.csv 2>&1
B="python bench.py --steps 1 --warmup 1 --no-sweep --no-e2e --no-cpu --no-configs --no-fp64 --nt 20"
$B > gpurun_out/b_o8.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:acoustic_queue -s 30 -c 2 --csv $B > gpurun_out/ncu_flops_o8.csv 2>&1
