# final validation of the build: every GPU test, smoke, every bench config + the reference arm, C2/C4 launch lists
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -4
python -c "import sys; sys.path.insert(0,'.'); import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -c 300 gpurun_out/bench_C2.json
for c in C4 C4D C3L C1 C2D C3 C3D; do timeout 1200 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 200 gpurun_out/bench_$c.json; done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; tail -c 200 gpurun_out/bench_ref.json
K='regex:router|perm|grouped|combine|small_ffn'
timeout 900 ncu --kernel-name "$K" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 24 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_c2.csv 2>/dev/null; python tools/launch_table.py gpurun_out/ncu_launches_c2.csv | tail -8
timeout 900 ncu --kernel-name "$K" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 30 --csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_c4.csv 2>/dev/null; python tools/launch_table.py gpurun_out/ncu_launches_c4.csv | tail -12
