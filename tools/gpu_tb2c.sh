timeout 200 python tools/time_orders.py --orders 4,8 --variants tb2 --nt 20 --tag default > gpurun_out/tb2c.log 2>&1
B200FD_LIB=build/tbw0/libb200fd.so timeout 200 python tools/time_orders.py --orders 4,8 --variants tb2 --nt 20 --tag tbw0 >> gpurun_out/tb2c.log 2>&1
cat gpurun_out/tb2c.log
bash tools/prof_tb2.sh default
bash tools/prof_tb2.sh tbw0
