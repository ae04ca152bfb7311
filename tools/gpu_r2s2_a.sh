set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -8
python -c "import sys; sys.path.insert(0,'.'); import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -c 2500 gpurun_out/bench_C2.json
for c in C4 C4D; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 900 gpurun_out/bench_$c.json; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_c4.csv 2>/dev/null; python tools/launch_table.py gpurun_out/ncu_launches_c4.csv | tail -30
