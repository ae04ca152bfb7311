# same-box A/B of two library builds (ablib/libcoxmoe_old.so vs the in-tree build) with the permute and combine stage times
for i in 1 2 3; do for lib in ablib/libcoxmoe_old.so paper_2605_17889_b200/libcoxmoe.so; do for c in ${CONFIGS:-C4 C2}; do
  COXMOE_LIB=$PWD/$lib timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']; print(\"$c $(basename $lib)\", round(d[\"value\"]/1e6,3), 'perm', round(s['permute'],3), 'comb', round(s['combine'],3), d[\"clocks\"][\"sm_mhz\"])"
done; done; done
