# ncu full captures of queue2 at orders 8 and 16 (after plain runs exit 0).
set -x
for o in 8 16; do
  python tools/prof_step.py --order $o --nt 6 --random --variant queue2 > gpurun_out/q2p$o.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:acoustic_queue2 -s 3 -c 1 -o gpurun_out/q2full_o$o python tools/prof_step.py --order $o --nt 6 --random --variant queue2 > gpurun_out/q2ncu$o.log 2>&1
  echo "o$o rc=$?"
done
