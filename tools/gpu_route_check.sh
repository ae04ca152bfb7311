# decode router: parity tests + A/B (run under gpurun)
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in C4D C2D; do for r in 1 0 1 0; do COX_ROUTER_DECODE=$r timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c router_decode=$r', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['gpu_launches'])"; done; done
timeout 600 python tools/sweep_decode.py 2>&1 | tail -10
