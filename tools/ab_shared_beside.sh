# shared-expert GEMMs beside the permute (run under gpurun)
for r in 1 0 1 0 1 0; do COX_SHARED_BESIDE=$r timeout 300 python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 beside=$r', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], d['stages_ms'])"; done
