set -x
timeout 1200 python -m pytest tests/test_gpu_router_e8.py tests/test_gpu_fullbatch.py tests/test_gpu_parity.py tests/test_gpu_ep.py -q -rf 2>&1 | tail -25
python tools/bench_router.py
COX_ROUTER=generic python tools/bench_router.py
bash tools/ab_l2.sh "X=1" "COX_L2_PERSIST_MB=64 COX_GEMM_L2_K4=1" "COX_L2_PERSIST_MB=64 COX_GEMM_L2_K4=2" "COX_L2_PERSIST_MB=80 COX_GEMM_L2_K3=2 COX_GEMM_BAND_K3=28 COX_GEMM_L2_K4=2" "COX_L2_PERSIST_MB=40 COX_GEMM_L2_K3=1 COX_GEMM_L2_K4=1 COX_GEMM_BAND_K4=4"
for v in "p64k4l1:COX_L2_PERSIST_MB=64 COX_GEMM_L2_K4=1" "p64k4l2:COX_L2_PERSIST_MB=64 COX_GEMM_L2_K4=2" "p80k3b28:COX_L2_PERSIST_MB=80 COX_GEMM_L2_K3=2 COX_GEMM_BAND_K3=28"; do bash tools/ncu_dram.sh "${v%%:*}" "${v#*:}"; done
timeout 600 python bench.py --no-e2e 2>&1 | tail -1 | cut -c1-900
