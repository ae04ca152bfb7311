# router changes: probe + parity tests + decode sweep points (run under gpurun)
./tools/probes/route_probe
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in C4D C2D; do for r in 0 1; do COX_DECODE_ROUTE_IN=$r timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c route_in=$r', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['stages_ms'])"; done; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', round(d['value']/1e6,4), d['stages_ms'])"
