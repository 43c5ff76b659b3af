# Source-level ncu capture of tti_pack on config 4 (one mid-run launch).
LIB=${1:-default}
if [ $LIB != default ]; then export B200FD_LIB=build/$LIB/libb200fd.so; fi
python tools/time_tti.py 6 > gpurun_out/tti_$LIB.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tti_pack -s 3 -c 1 \
  -o gpurun_out/tti_$LIB python tools/time_tti.py 6 > gpurun_out/ncu_tti_$LIB.log 2>&1
echo "ncu rc=$?"; cat gpurun_out/tti_$LIB.log
