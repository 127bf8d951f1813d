export BENCH_EXTRA="--no-e2e"
bash scratch/variants.sh base: win3:-DTCMIS_SEL_WIN=3 win4:-DTCMIS_SEL_WIN=4 win3m6:"-DTCMIS_SEL_WIN=3 -DTCMIS_SEL_MINB=6" base2: -- rmat22 rmat26 grid rgg > gpurun_out/variants_win.txt 2>&1
