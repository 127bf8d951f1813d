# build + bench each variant given as NAME:FLAGS ... -- configs
specs=(); while [ "$1" != "--" ]; do specs+=("$1"); shift; done; shift
for spec in "${specs[@]}"; do
  name=${spec%%:*}; flags=${spec#*:}
  touch paper_2605_29604_b200/csrc/select.cuh
  TCMIS_NVCC_EXTRA="$flags" python -m paper_2605_29604_b200.build > /dev/null 2>&1
  echo "== $name $flags"
  bash scratch/ab.sh "$@"
done
