# Full ncu captures of the remaining round-2 production kernels (elastic passes, acoustic
# orders 12 and 16) and of the experimental el_fused kernel; each after a plain run exited 0.
N="ncu --set full --clock-control none --import-source on"
python tools/time_elastic.py 4 > gpurun_out/el4.log 2>&1 && \
  $N -k regex:el_queue -s 4 -c 2 -o gpurun_out/full_el python tools/time_elastic.py 4 > gpurun_out/ncu_el.log 2>&1
B200FD_EL_FUSE=4 python tools/el_window_probe.py 2 > gpurun_out/elf2.log 2>&1 && \
  B200FD_EL_FUSE=4 $N --cache-control none -k regex:el_fused -s 4 -c 1 -o gpurun_out/full_elfused python tools/el_window_probe.py 2 > gpurun_out/ncu_elf.log 2>&1
for o in 12 16; do
  python tools/time_orders.py --orders $o --nt 6 > gpurun_out/o$o.log 2>&1 && \
    $N -k regex:acoustic_queue -s 4 -c 1 -o gpurun_out/full_o$o python tools/time_orders.py --orders $o --nt 6 > gpurun_out/ncu_o$o.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
# summarise on the box (the reports together exceed gpurun's 64 MiB return limit)
for r in el elfused o12 o16; do
  (python tools/ncu_summary.py gpurun_out/full_$r.ncu-rep; python tools/ncu_src_stalls.py gpurun_out/full_$r.ncu-rep) > gpurun_out/r02_ncu_full_$r.txt 2>&1
done
rm -f gpurun_out/full_el.ncu-rep gpurun_out/full_o12.ncu-rep gpurun_out/full_o16.ncu-rep
