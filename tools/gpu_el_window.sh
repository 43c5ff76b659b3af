# Windowed elastic schedule: time and bit-compare against the two full passes,
# then DRAM bytes per step from ncu (no cache flush between kernels).
O=gpurun_out/el_window.jsonl; : > $O
python tools/el_window_probe.py 30 >> $O 2>gpurun_out/el_window.err
for C in 4 6 8 12 16 32; do
  B200FD_EL_WINDOW=$C python tools/el_window_probe.py 30 >> $O 2>>gpurun_out/el_window.err
  B200FD_EL_WINDOW=$C B200FD_EL_WINDOW_STREAMS=2 python tools/el_window_probe.py 30 >> $O 2>>gpurun_out/el_window.err
done
for C in 8 16; do
  B200FD_EL_WINDOW=$C B200FD_EL_WINDOW_STREAMS=2 B200FD_EL_WINDOW_LEAD=2 python tools/el_window_probe.py 30 >> $O 2>>gpurun_out/el_window.err
  B200FD_EL_WINDOW=$C B200FD_EL_WINDOW_STREAMS=2 B200FD_EL_WINDOW_LEAD=4 python tools/el_window_probe.py 30 >> $O 2>>gpurun_out/el_window.err
done
cat $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for C in 0 4 8 16; do
  B200FD_EL_WINDOW=$C ncu --metrics $M --clock-control none --cache-control none -k regex:el_queue --csv \
    python tools/el_window_probe.py 1 > gpurun_out/el_window_ncu_$C.csv 2>&1
  python - $C <<'PY'
import csv, sys
C = sys.argv[1]
rows = list(csv.reader(l for l in open(f"gpurun_out/el_window_ncu_{C}.csv", errors="replace") if l.startswith('"')))
hdr = rows[0]; iN = hdr.index("Metric Name"); iV = hdr.index("Metric Value"); iU = hdr.index("Metric Unit")
tot = {}
n = 0
for r in rows[1:]:
    v = float(r[iV].replace(",", ""))
    u = r[iU]
    if u == "Gbyte": v *= 1e9
    elif u == "Mbyte": v *= 1e6
    elif u == "Kbyte": v *= 1e3
    tot[r[iN]] = tot.get(r[iN], 0.0) + v
    n += 1
steps = 13  # 12 hashed + 1 timed
pts = 320 ** 3 * steps
print(C, "launches", n // 3, "B/pt read", round(tot["dram__bytes_read.sum"] / pts, 2), "write",
      round(tot["dram__bytes_write.sum"] / pts, 2))
PY
done
