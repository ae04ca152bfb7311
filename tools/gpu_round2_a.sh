set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import sys; sys.path.insert(0,'.'); import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
bash tools/ab_l2.sh "X=1" "COX_GEMM_L2_K4=1" "COX_GEMM_L2_K4=2" "COX_GEMM_L2_K3=1 COX_GEMM_BAND_K3=28" "COX_GEMM_L2_K3=2 COX_GEMM_BAND_K3=28" "COX_GEMM_L2_K4=1 COX_GEMM_BAND_K4=16" 2>&1
for v in "base:X=1" "k4l1:COX_GEMM_L2_K4=1" "k4l2:COX_GEMM_L2_K4=2" "k3l1b28:COX_GEMM_L2_K3=1 COX_GEMM_BAND_K3=28"; do bash tools/ncu_dram.sh "${v%%:*}" "${v#*:}"; done
timeout 600 python bench.py 2>&1 | tail -2
