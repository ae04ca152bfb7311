timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stack.py -q -x -rf 2>&1 | tail -3
timeout 600 python tools/c4_order.py ablate C4
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:router_rescore --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_rescore2_c4 python tools/bench_router.py > /dev/null 2>&1; ls -la gpurun_out/*.ncu-rep
