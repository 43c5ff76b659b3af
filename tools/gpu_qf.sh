S="timeout 300 python tools/queue_stress.py --order 2 --reps 7"
{
$S --tag default
B200FD_LIB=build/qf1/libb200fd.so $S --tag qf1
B200FD_LIB=build/qf2/libb200fd.so $S --tag qf2
} > gpurun_out/qf.log 2>&1
grep -v "^  rep" gpurun_out/qf.log
