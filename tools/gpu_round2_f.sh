set -x
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -8
python -c "import sys; sys.path.insert(0,'.'); import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -c 2500 gpurun_out/bench_C2.json
for c in C1 C3L C4 C4D C2D; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 600 gpurun_out/bench_$c.json; done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; tail -c 400 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_c2.csv 2>/dev/null; wc -l gpurun_out/ncu_launches_c2.csv
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:router_e8 --launch-skip 3 --launch-count 1 -o gpurun_out/ncu_router_e8_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls -la gpurun_out/*.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:grouped_gemm --launch-skip 6 --launch-count 2 -o gpurun_out/ncu_gemm_c4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls -la gpurun_out/*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_c4.csv 2>/dev/null; wc -l gpurun_out/ncu_launches_c4.csv
