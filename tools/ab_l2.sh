#!/bin/bash
# L2 cache-policy / raster-band A/B of the prefill grouped GEMMs (run under gpurun):
#   bash tools/ab_l2.sh "<env settings> ..."   each argument one variant, e.g. "COX_GEMM_L2_K4=1"
run() { env $1 timeout 300 python bench.py --config ${CFG:-C2} --no-cpu-baseline --no-e2e --steps ${STEPS:-10} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${CFG:-C2}', '$1', round(d['value']/1e6,4), 'M k3', round(r['k3_ms'],2), 'k4', round(r['k4_ms'],2), 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w_max'), flush=True)"; }
for rep in 1 2; do for a in "$@"; do run "$a"; done; done
