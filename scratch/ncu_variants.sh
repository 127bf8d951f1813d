# ncu --set full on round-1 k_select for each variant NAME:FLAGS
cfg=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  touch paper_2605_29604_b200/csrc/select.cuh
  TCMIS_NVCC_EXTRA="$flags" python -m paper_2605_29604_b200.build > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_select$|k_select\(' -s 0 -c 1 -o gpurun_out/sel_${cfg}_${name} python scratch/ncu_target.py $cfg > gpurun_out/ncu_${name}.log 2>&1
  tail -1 gpurun_out/ncu_${name}.log
done
