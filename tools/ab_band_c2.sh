run() { env "$@" timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']/1e6,4), 'M k3', round(d['roofline']['k3_ms'],2), 'k4', round(d['roofline']['k4_ms'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"; }
run X=1
run COX_GEMM_BAND_K4=4
run COX_GEMM_BAND_K4=16
run COX_GEMM_BAND_K3=8
run COX_GEMM_BAND_K3=28
run X=1
run COX_GEMM_BAND_K4=4
