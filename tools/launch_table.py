"""Summarise an ncu --csv launch list (tools/gpu_round2_g.sh) as one line per kernel launch."""
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
by = {}
for r in rows[1:]:
    by.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = r[vi]
tot = 0.0
for k, v in sorted(by.items()):
    t = float(v.get("gpu__time_duration.sum", "0").replace(",", ""))
    tot += t
    extra = v.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", v.get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", ""))
    print(f"{k:3d} {v['k'][:60]:60s} {t / 1e3:9.1f} us  rd {float(v.get('dram__bytes_read.sum', '0')) / 1e9:7.3f} GB"
          f"  wr {float(v.get('dram__bytes_write.sum', '0')) / 1e9:7.3f} GB  {extra}")
print(f"total {tot / 1e6:.3f} ms")
