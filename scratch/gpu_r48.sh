bash scratch/ncu_kernel.sh grid 'k_probe_select' ncu_probe_grid_r2 4
bash scratch/ncu_kernel.sh grid 'k_probe_select' ncu_probe_grid_r1 3
