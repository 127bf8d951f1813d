bash scratch/variants.sh "tm32:" "tm64:-DTCMIS_THREAD_MAX=64" "tm16:-DTCMIS_THREAD_MAX=16" "tm128:-DTCMIS_THREAD_MAX=128" -- rmat22 rmat26 grid > gpurun_out/variants_tm.txt 2>&1
