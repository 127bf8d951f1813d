set -x
TCMIS_TAIL_THRESHOLD=0 bash scratch/ab.sh rmat22 er grid > gpurun_out/ab_notail.txt 2>&1
bash scratch/ab.sh rmat22 er grid > gpurun_out/ab_tail.txt 2>&1
