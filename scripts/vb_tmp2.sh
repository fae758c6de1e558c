bash scripts/ncu_kernel.sh k3g "k_guard_points" 5 1
