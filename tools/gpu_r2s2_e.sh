timeout 1200 python -m pytest tests/test_gpu_router_tc.py tests/test_gpu_fullbatch.py tests/test_gpu_robust.py tests/test_gpu_parity.py -q -x -rf 2>&1 | tail -5
python tools/bench_router.py
