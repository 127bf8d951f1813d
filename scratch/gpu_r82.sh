python -m paper_2605_29604_b200.build > /dev/null 2>&1
bash scratch/ncu_kernel.sh rmat26 'k_select$' full_select4_rmat26 0
