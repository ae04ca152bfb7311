# round-end bench lines for every config (run under gpurun): gpurun_out/fin_<cfg>.json
for c in C2 C4 C4D C2D C1 C3L; do timeout 900 python bench.py --config $c > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; done
timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
