# K per stage / ring depth A/B for the grouped GEMMs (run under gpurun)
run() { env "$@" timeout 300 python bench.py --config ${CFG:-C4} --no-cpu-baseline --no-e2e --steps ${STEPS:-20} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${CFG:-C4}', '$*', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],2), 'ms k3', round(d['roofline']['k3_ms'],2), 'k4', round(d['roofline']['k4_ms'],2), d['clocks']['sm_mhz'])"; }
run X=1
run COX_GEMM_BK=64 COX_GEMM_NOSTG=1
run X=1
run COX_GEMM_BK=64 COX_GEMM_NOSTG=1
CFG=C2 STEPS=10 run X=1
CFG=C2 STEPS=10 run COX_GEMM_BK=64 COX_GEMM_NOSTG=1
CFG=C2 STEPS=10 run COX_GEMM_NOSTG=1
