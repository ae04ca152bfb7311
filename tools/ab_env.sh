# Same-box A/B of environment switches for one config (run under gpurun):
#   CFG=C2 bash tools/ab_env.sh "X=1" "COX_GEMM_L2_K4=1"
run() { env $1 timeout 300 python bench.py --config ${CFG:-C2} --no-cpu-baseline --no-e2e --steps ${STEPS:-15} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${CFG:-C2}', '$1', round(d['value']/1e6,4), 'M', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"; }
for rep in 1 2; do for a in "$@"; do run "$a"; done; done
