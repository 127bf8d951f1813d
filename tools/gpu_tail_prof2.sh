mkdir -p gpurun_out
rm -f paper_2605_29604_b200/_obj/solver.cu.o
TCMIS_NVCC_EXTRA=-DTCMIS_TAIL_PROF python -m paper_2605_29604_b200.build > /dev/null 2>&1
for c in rmat22 er; do timeout 600 python tools/tail_prof.py $c > gpurun_out/tail_prof_$c.txt 2>&1; tail -14 gpurun_out/tail_prof_$c.txt; done
ORDER=none timeout 600 python tools/tail_prof.py rmat22 > gpurun_out/tail_prof_rmat22_none.txt 2>&1; tail -14 gpurun_out/tail_prof_rmat22_none.txt
