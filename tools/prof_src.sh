# Source-level ncu captures of the acoustic queue kernel (one mid-run launch per order).
set -x
for o in ${ORDERS:-8 16}; do
  python tools/prof_step.py --order $o --random --nt 6 > gpurun_out/p$o.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:acoustic_queue -s 3 -c 1 \
      -o gpurun_out/src_o$o python tools/prof_step.py --order $o --random --nt 6 > gpurun_out/ncu_o$o.log 2>&1
done
ls -la gpurun_out
