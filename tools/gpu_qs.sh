S="timeout 300 python tools/queue_stress.py --reps 5"
{
$S --order 4
$S --order 6
$S --order 2 --nosponge
$S --order 2 --norec
$S --order 2 --nosrc
$S --order 2 --scalarm
$S --order 2 --variant direct --reps 3
} > gpurun_out/qs2.log 2>&1
grep -v "^  rep" gpurun_out/qs2.log
