set -x
timeout 900 python -m pytest tests/test_gpu_stack.py -q -rf 2>&1 | tail -15
timeout 300 python tools/bench_fetch.py
timeout 1200 python bench.py --config C3D 2>&1 | tail -3
timeout 1500 python bench.py --config C3 2>&1 | tail -3
