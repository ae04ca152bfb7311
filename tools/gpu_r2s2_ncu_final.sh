# ncu --set full of every hot kernel of the final build (one launch each), for profiles/r02/final
set -x
O=gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:"router_e8|perm_copy|grouped_gemm|combine_kernel" --launch-skip 8 --launch-count 5 -o $O/ncu_final_c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:"router_screen|router_rescore|perm_copy|grouped_gemm|combine_kernel" --launch-skip 14 --launch-count 8 -o $O/ncu_final_c4 -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"router_decode|small_ffn" --launch-skip 20 --launch-count 2 -o $O/ncu_final_c4d -f python bench.py --config C4D --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $O/*.ncu-rep
