# Queue kernel x-chunk count A/B at 512^3 (default heuristic vs fixed counts).
for c in 0 1 2 4 8 16; do
  if [ $c = 0 ]; then unset B200FD_QCHUNKS; else export B200FD_QCHUNKS=$c; fi
  timeout 300 python tools/time_orders.py --orders 4,8,16 --variants queue --nt 30 --tag chunks$c
done > gpurun_out/chunks.log 2>&1
cat gpurun_out/chunks.log
