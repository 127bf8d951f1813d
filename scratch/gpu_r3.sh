# L2 hint variants (rebuilt on the box), then default build: parity + tile-form benches
set -x
bash scratch/variants.sh "both:" "nopersist:-DTCMIS_NO_L2_PERSIST" "nostream:-DTCMIS_STREAM_HINTS=0" "neither:-DTCMIS_NO_L2_PERSIST -DTCMIS_STREAM_HINTS=0" -- rgg rmat22 grid > gpurun_out/variants.txt 2>&1
touch paper_2605_29604_b200/csrc/select.cuh
python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for ex in tile-bits tile-mma pull push; do echo "== $ex"; BENCH_EXTRA="--exclusion $ex" bash scratch/ab.sh grid rmat22; done > gpurun_out/excl_forms.txt 2>&1
