touch paper_2605_29604_b200/csrc/select.cuh
TCMIS_NVCC_EXTRA="-DTCMIS_TAIL_PROF" python -m paper_2605_29604_b200.build > /dev/null 2>&1
python scratch/tail_prof.py er grid rmat22 rmat26 > gpurun_out/tail_prof.txt 2>&1
