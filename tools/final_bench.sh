# round-end checks (run under gpurun): GPU tests, smoke, bench lines -> gpurun_out/fin_<cfg>.json
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/fin_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/fin_smoke.log
for c in ${FIN_CONFIGS:-C2 C4D C4}; do timeout 900 python bench.py --config $c > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; done
