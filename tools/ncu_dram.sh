#!/bin/bash
# DRAM bytes + duration per grouped-GEMM launch under ncu for one env variant (run under gpurun):
#   bash tools/ncu_dram.sh <tag> "<env settings>"
tag=$1; shift
env $1 timeout 900 ncu --kernel-name regex:grouped_gemm --launch-skip 2 --launch-count 2 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
  --clock-control none --csv python bench.py --config ${CFG:-C2} --no-cpu-baseline --no-e2e --steps 1 --warmup 3 \
  > gpurun_out/ncu_dram_${tag}.csv 2> gpurun_out/ncu_dram_${tag}.err
python - "$tag" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = list(csv.reader(l for l in open(f"gpurun_out/ncu_dram_{tag}.csv") if l.startswith('"')))
h = rows[0]; out = {}
for r in rows[1:]:
    d = dict(zip(h, r)); key = (d["ID"], d["Kernel Name"][:40])
    out.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
for (i, n), m in out.items():
    print(tag, i, n, {k.split("__")[1]: v for k, v in m.items()})
PY
