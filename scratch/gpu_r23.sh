set -x
bash scratch/ncu_kernel.sh rgg 'k_probe_select' ncu_probe_rgg 3
bash scratch/ncu_kernel.sh rmat26 'k_select\(' ncu_select_rmat26 2
bash scratch/ncu_kernel.sh rmat22 'k_select\(' ncu_select_rmat22 1
bash scratch/ncu_kernel.sh rmat22 'k_probe_select' ncu_probe_rmat22 1
bash scratch/ncu_kernel.sh rmat22 'k_round_end' ncu_roundend_rmat22 1
