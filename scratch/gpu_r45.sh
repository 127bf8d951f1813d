set -x
bash scratch/variants.sh "u16b1:" "u8b2:-DTCMIS_TAIL_UNROLL=8 -DTCMIS_TAIL_MINB=2" "u4b2:-DTCMIS_TAIL_UNROLL=4 -DTCMIS_TAIL_MINB=2" -- rmat22 er grid rgg > gpurun_out/variants_tailocc.txt 2>&1
