set -x
timeout 600 python tools/c4_order.py 3 10
python tools/bench_router.py
K='regex:router|perm|grouped|combine'
timeout 900 ncu --kernel-name "$K" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -c 40 --csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_c4.csv 2>/dev/null; python tools/launch_table.py gpurun_out/ncu_launches_c4.csv | tail -25
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:router_rescore --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_rescore_c4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls -la gpurun_out/*.ncu-rep
