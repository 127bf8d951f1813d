export BENCH_EXTRA="--no-e2e"
bash scratch/variants.sh base: win1:-DTCMIS_SEL_WIN=1 base2: -- rmat26 rmat22 > gpurun_out/variants_win1.txt 2>&1
