set -x
bash scratch/variants.sh "hints:" "nohints:-DTCMIS_STREAM_HINTS=0" -- rgg rmat22 grid > gpurun_out/variants.txt 2>&1
touch paper_2605_29604_b200/csrc/select.cuh
python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for ex in tile-bits tile-mma; do echo "== $ex"; BENCH_EXTRA="--exclusion $ex" bash scratch/ab.sh grid rmat22 rgg; done > gpurun_out/excl_forms.txt 2>&1
# ncu --set full: round-1 exclusion kernels of every form on grid and rmat22 (skip 1 = second solve)
for c in grid rmat22; do
  EXCL=tile-bits bash scratch/ncu_kernel.sh $c 'k_tile_excl_bits' excl_bits_$c 3
  EXCL=tile-mma bash scratch/ncu_kernel.sh $c 'k_tile_excl_mma' excl_mma_$c 3
  EXCL=pull bash scratch/ncu_kernel.sh $c 'k_probe_pull' excl_probepull_$c 3
  EXCL=pull bash scratch/ncu_kernel.sh $c 'k_update_pull' excl_updpull_$c 3
  EXCL=push bash scratch/ncu_kernel.sh $c 'k_update\b|k_update\(' excl_update_$c 3
done
bash scratch/ncu_kernel.sh rmat22 'k_priorities' full_prio_rmat22 1
