# L2 evict_first on the decode weight stream: A/B + trace (run under gpurun)
run() { COXMOE_LIB=ablib/$1.so timeout 300 python bench.py --config $2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"; }
for c in C4D C2D; do run new $c; run noevict $c; run new $c; run noevict $c; done
TRACE_GRAPH=1 timeout 300 python tools/trace_small.py --run-only C4D C2D 2>&1 | grep "^\["
timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_decode_routed.py -q -x 2>&1 | tail -1
