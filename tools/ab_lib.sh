# A/B of two library builds on the same box (run under gpurun): ablib/<name>.so
run() { COXMOE_LIB=ablib/$1.so timeout 300 python bench.py --config $2 --no-cpu-baseline --no-e2e --steps ${3:-20} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],3), 'ms k3', round(d['roofline'].get('k3_ms') or 0,3), 'k4', round(d['roofline'].get('k4_ms') or 0,3), d['clocks']['sm_mhz'])"; }
for c in C1 C4 C3L; do run relaxed $c; run silufast $c; done
run relaxed C2 10; run silufast C2 10; run relaxed C2 10; run silufast C2 10
