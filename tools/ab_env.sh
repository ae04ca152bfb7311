#!/bin/bash
# A/B an environment switch on the same build: tools/ab_env.sh VAR "valA valB" [bench args...]
VAR=$1; VALS=$2; shift 2
for i in 1 2; do
  for v in $VALS; do
    env $VAR=$v python bench.py --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']
print('$VAR=$v', round(j['value']), 'k3', round(r.get('k3_ms') or 0,2), 'k4', round(r.get('k4_ms') or 0,2), 'mhz', j['clocks']['sm_mhz'], 'W', j['clocks'].get('power_w_max'))"
  done
done
