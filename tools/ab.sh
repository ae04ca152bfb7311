#!/bin/bash
# A/B two builds of libcoxmoe on the same GPU box: tools/ab.sh <libA> <libB> [bench args...]
A=$1; B=$2; shift 2
for i in 1 2; do
  for L in $A $B; do
    COXMOE_LIB=$L python bench.py --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']
print('$L'.split('/')[-1], round(j['value']), 'k3', round(r['k3_ms'],2), 'k4', round(r['k4_ms'],2), 'mhz', j['clocks']['sm_mhz'], j['stages_ms'])"
  done
done
