set -x
timeout 1200 python -m pytest tests/test_gpu_router_tc.py tests/test_gpu_fullbatch.py tests/test_gpu_parity.py tests/test_gpu_robust.py -q -rf 2>&1 | tail -5
python tools/bench_router.py
K='regex:router|perm'
timeout 900 ncu --kernel-name "$K" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_c4_router.csv 2>/dev/null; python tools/launch_table.py gpurun_out/ncu_launches_c4_router.csv
for i in 1 2; do timeout 900 python bench.py --config C4 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],2), d['stages_ms'], d['clocks']['sm_mhz'])"; done
