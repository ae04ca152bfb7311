#!/usr/bin/env python
"""Summarise an ncu report (raw page) into a compact per-kernel table (markdown + JSON).

    python tools/ncu_summary.py gpurun_out/r01_c2_full.ncu-rep > profiles/r01/ncu_c2.md
"""
import csv
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clk"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_lsb"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for m, short in METRICS:
            if m in hdr:
                i = hdr.index(m)
                rec[short] = f"{r[i]} {units[i]}".strip()
        recs.append(rec)
    cols = ["kernel"] + [s for _, s in METRICS]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for rec in recs:
        print("| " + " | ".join(rec.get(c, "") for c in cols) + " |")
    print()
    print("```json")
    print(json.dumps(recs, indent=1))
    print("```")


if __name__ == "__main__":
    main(sys.argv[1])
