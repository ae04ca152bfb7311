# evidence sweeps on the final build: batch-size sweep (decode -> prefill), the
# paper's coalesced-vs-micro-batched ablation, repeated headline lines
set -x
timeout 1200 python tools/sweep_tokens.py C4 > gpurun_out/sweep_tokens_c4.txt 2>&1; cat gpurun_out/sweep_tokens_c4.txt
timeout 1800 python tools/sweep_tokens.py C2 > gpurun_out/sweep_tokens_c2.txt 2>&1; cat gpurun_out/sweep_tokens_c2.txt
for mb in 4096 16384 65536; do timeout 900 python bench.py --microbatch $mb --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_mb$mb.json 2>&1; tail -c 300 gpurun_out/bench_c2_mb$mb.json; done
for i in 1 2; do for c in C2 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e | tail -1 > gpurun_out/bench_rep_${c}_$i.json; tail -c 250 gpurun_out/bench_rep_${c}_$i.json; done; done
