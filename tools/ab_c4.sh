run() { env "$@" timeout 300 python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],2), 'ms k3', round(d['roofline']['k3_ms'],2), 'k4', round(d['roofline']['k4_ms'],2), d['clocks']['sm_mhz'])"; }
run X=1
run COX_GEMM_BK=64
run COX_GEMM_BK=128
run X=1
run COX_GEMM_BK=64
