set -x
bash scratch/variants.sh "s128_l512:" "s128_l2048:-DTCMIS_TAIL_LONG=2048" "s0_l512:-DTCMIS_TAIL_SMALL=0" "s0_linf:-DTCMIS_TAIL_SMALL=0 -DTCMIS_TAIL_LONG=1000000000" "s32_l1024:-DTCMIS_TAIL_SMALL=32 -DTCMIS_TAIL_LONG=1024" -- rmat22 er grid > gpurun_out/variants_tail.txt 2>&1
