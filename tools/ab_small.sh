# decode A/B (run under gpurun): C4D step time
run() { env "$@" timeout 120 python bench.py --config C4D --no-cpu-baseline --no-e2e --steps 3000 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['gpu_launches'])"; }
run COX_ROUTER_DECODE=1
run COX_ROUTER_DECODE=0
run COX_ROUTER_DECODE=1
run COX_ROUTER_DECODE=0
