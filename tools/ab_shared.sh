# A/B of the fused shared-down + combine epilogue (run under gpurun): ablib/<name>.so
run() { COXMOE_LIB=ablib/$1.so timeout 300 python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$1 $2', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in s.items()}, d['clocks']['sm_mhz'])"; }
timeout 300 python -m pytest tests/test_gpu_shared_combine.py -q -x 2>&1 | tail -1
for n in u2 u4; do run $n; done
COX_SHARED_FUSE=0 run u4 unfused
for n in u2 u4; do run $n; done
