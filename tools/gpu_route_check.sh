# router changes: parity tests + decode trace + C4D/C2D bench (run under gpurun)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_router_tc.py tests/test_gpu_small.py tests/test_gpu_decode_routed.py tests/test_gpu_robust.py -q -x 2>&1 | tail -2
TRACE_GRAPH=1 timeout 300 python tools/trace_small.py --run-only C4D C2D 2>&1 | grep "^\["
for c in C4D C2D; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"; done
