set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash scratch/variants.sh "g8:" "g4:-DTCMIS_TAIL_GROUP=4" "g16:-DTCMIS_TAIL_GROUP=16" "g4u8:-DTCMIS_TAIL_GROUP=4 -DTCMIS_TAIL_UNROLL=8" -- rmat22 er grid rgg > gpurun_out/variants_group.txt 2>&1
