set -x
bash scratch/variants.sh "br8k:" "br2k:-DTCMIS_BLOCK_ROW=2048" "broff:-DTCMIS_BLOCK_ROW=2000000000" -- rmat22 rmat26 > gpurun_out/variants_br.txt 2>&1
touch paper_2605_29604_b200/csrc/select.cuh; python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
