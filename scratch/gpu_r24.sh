set -x
bash scratch/variants.sh "hint:" "nohint:-DTCMIS_GATHER_HINT=0" -- rgg rmat22 grid rmat26 > gpurun_out/variants_hint.txt 2>&1
touch paper_2605_29604_b200/csrc/select.cuh; python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash scratch/ncu_kernel.sh rgg 'k_probe_select' ncu_probe_rgg2 3
bash scratch/ncu_kernel.sh rmat26 '^k_select$' ncu_select_rmat26 2
bash scratch/ncu_kernel.sh rmat22 'k_select$' ncu_select_rmat22 1
