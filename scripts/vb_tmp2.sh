bash scripts/ncu_kernel.sh fin "k_finalize" 5 1
