# Fused elastic step (el_fused): bit-compare against the two full passes, time,
# DRAM bytes per point.  Short wait bound so a scheduling bug cannot hang the box.
export B200FD_WAIT_CYCLES=$((1<<25))
O=gpurun_out/el_fuse.jsonl; : > $O
timeout 300 python tools/el_window_probe.py 30 >> $O 2>gpurun_out/el_fuse.err
for C in 4 5 6 8; do
  B200FD_EL_FUSE=$C timeout 300 python tools/el_window_probe.py 30 >> $O 2>>gpurun_out/el_fuse.err
done
for L in 40 100 200; do
  B200FD_EL_FUSE=4 B200FD_EL_FUSE_LAG=$L timeout 300 python tools/el_window_probe.py 30 >> $O 2>>gpurun_out/el_fuse.err
done
cat $O; tail -5 gpurun_out/el_fuse.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for C in 4 6; do
  B200FD_EL_FUSE=$C timeout 600 ncu --metrics $M --clock-control none --cache-control none -k regex:el_fused --csv \
    python tools/el_window_probe.py 1 > gpurun_out/el_fuse_ncu_$C.csv 2>&1
  python - $C <<'PY'
import csv, sys
C = sys.argv[1]
rows = list(csv.reader(l for l in open(f"gpurun_out/el_fuse_ncu_{C}.csv", errors="replace") if l.startswith('"')))
hdr = rows[0]; iN = hdr.index("Metric Name"); iV = hdr.index("Metric Value"); iU = hdr.index("Metric Unit")
tot = {}; n = 0
for r in rows[1:]:
    v = float(r[iV].replace(",", "")); u = r[iU]
    v *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}.get(u, 1.0)
    tot[r[iN]] = tot.get(r[iN], 0.0) + v; n += 1
pts = 320 ** 3 * (n // 3)
print("fuse", C, "launches", n // 3, "B/pt read", round(tot["dram__bytes_read.sum"] / pts, 2), "write",
      round(tot["dram__bytes_write.sum"] / pts, 2), "us/launch", round(tot["gpu__time_duration.sum"] / (n // 3) / (1e3 if True else 1), 1))
PY
done
