TCMIS_NVCC_EXTRA="-DTCMIS_PDL=1" python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pdl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pdl.log
bash scratch/variants.sh base: pdl:-DTCMIS_PDL=1 base2: pdl2:-DTCMIS_PDL=1 -- rmat22 grid rgg er > gpurun_out/variants_pdl.txt 2>&1
