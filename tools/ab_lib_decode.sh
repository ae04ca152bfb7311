# decode A/B of two builds (ablib/<a>.so vs ablib/<b>.so) on the same box
run() { COXMOE_LIB=ablib/$1.so timeout 120 python bench.py --config C4D --no-cpu-baseline --no-e2e --steps 3000 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; }
for i in 1 2; do run $1; run $2; done
