# A/B of two library builds on the decode configs (run under gpurun): ablib/<name>.so
run() { COXMOE_LIB=ablib/$1.so timeout 300 python bench.py --config $2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; }
for c in C4D C2D; do run base $c; run new $c; run base $c; run new $c; done
