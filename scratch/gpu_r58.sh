python -m paper_2605_29604_b200.build > /dev/null 2>&1
bash scratch/ncu_kernel.sh rmat26 'k_select$' full_select_rmat26 1
bash scratch/ncu_kernel.sh rmat26 'k_update_pull' full_update_pull_rmat26 1
bash scratch/variants.sh base: hints0:-DTCMIS_STREAM_HINTS=0 ghint0:-DTCMIS_GATHER_HINT=0 base2: -- rmat26 > gpurun_out/variants_r58.txt 2>&1
