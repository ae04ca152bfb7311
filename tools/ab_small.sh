# Decode-path A/B on C4D (run under gpurun): step time for each environment
# setting, e.g. COX_SMALL_FROM_IDX=0 (router + permute + expert launch),
# COX_DECODE_DENSE=0, COX_PDL=0, COX_SMALL_VARIANT=1,64.
run() { env "$@" timeout 120 python bench.py --config C4D --no-cpu-baseline --no-e2e --steps 3000 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['gpu_launches'])"; }
run X=1
run COX_SMALL_FROM_IDX=0
run COX_PDL=0
