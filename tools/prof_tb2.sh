# ncu capture of one two-step launch (order 8, 512^3) for a given library.
LIB=${1:-default}
if [ $LIB != default ]; then export B200FD_LIB=build/$LIB/libb200fd.so; fi
timeout 300 ncu --set full --clock-control none --import-source on -k regex:acoustic_tb2 -s 2 -c 1 \
  -o gpurun_out/tb2_$LIB python tools/time_orders.py --orders 8 --variants tb2 --nt 6 > gpurun_out/ncu_tb2_$LIB.log 2>&1
echo "ncu rc=$?"
