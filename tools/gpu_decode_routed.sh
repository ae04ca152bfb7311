timeout 300 python -m pytest tests/test_gpu_decode_routed.py -q -x > gpurun_out/dr.log 2>&1
echo "exit $?" >> gpurun_out/dr.log
if grep -q "passed" gpurun_out/dr.log && ! grep -q "failed" gpurun_out/dr.log; then
  timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py -q -x > gpurun_out/dr2.log 2>&1
  for c in C4D C2D; do
    for r in 1 0 1 0; do
      COX_DECODE_ROUTE_IN=$r timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c route_in=$r', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['gpu_launches'], d['clocks']['sm_mhz'])" >> gpurun_out/dr_bench.log
    done
  done
fi
