# route_in prologue: A/B of library variants on C4D (run under gpurun)
run() { COXMOE_LIB=ablib/$1.so timeout 300 python bench.py --config C4D --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"; }
run new; run nopdl; run new; run nopdl
COX_DECODE_ROUTE_IN=0 run new
