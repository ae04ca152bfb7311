#!/bin/bash
# Raster-band sweep on one box: tools/band.sh "<k3 bands>" "<k4 bands>"
for b3 in $1; do for b4 in $2; do
  COX_GEMM_BAND_K3=$b3 COX_GEMM_BAND_K4=$b4 python bench.py --no-cpu-baseline --no-e2e --steps 6 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']
print('k3band $b3 k4band $b4', round(j['value']), 'k3', round(r['k3_ms'],2), 'k4', round(r['k4_ms'],2), 'mhz', j['clocks']['sm_mhz'], 'W', j['clocks'].get('power_w_max'))"
done; done
