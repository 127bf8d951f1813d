# tcgen05 Phase-1 tile product: parity, A/B against the CUDA-core tile form and CSR, ncu pages
mkdir -p gpurun_out/umma
timeout 900 python -m pytest tests/test_gpu_tile_cand.py -x -q > gpurun_out/umma/pytest.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/umma/pytest.txt
for spec in "grid csr" "grid tile" "grid tile-umma" "rgg_spatial_ids csr" "rgg_spatial_ids tile" "rgg_spatial_ids tile-umma"; do
  set -- $spec
  timeout 240 python bench.py --config $1 --candidates $2 --order none --no-e2e --no-cpu-baseline --no-k1 > gpurun_out/umma/tc_$1_$2.json 2> gpurun_out/umma/tc_$1_$2.log; echo "$1 $2 rc=$?"
  python - "$1" "$2" <<'P'
import json, sys
from collections import defaultdict
c, o = sys.argv[1:3]
d = json.loads(open(f'gpurun_out/umma/tc_{c}_{o}.json').read().strip().splitlines()[-1])
r1 = sorted([k for k in d['kernels_ms'] if k[1] == 1 and k[2] > 0.0068], key=lambda k: -k[2])
per = defaultdict(float)
for k, rd, ms in d['kernels_ms']: per[rd] += ms
print(c, o, d['device_resident']['ms'], d['config']['tile_cand_build'], dict((k, round(v, 4)) for k, v in sorted(per.items())), r1)
P
done
for c in grid rgg_spatial_ids; do
  for k in "k_tile_umma:umma:tile-umma" "k_tile_excl_bits:bits:tile"; do
    rx=$(echo $k | cut -d: -f1); nm=$(echo $k | cut -d: -f2); cand=$(echo $k | cut -d: -f3)
    CAND=$cand timeout 600 ncu --set full --clock-control none -k regex:"$rx" -s 1 -c 1 -o gpurun_out/umma/full_cand_${nm}_$c python tools/ncu_target.py $c > gpurun_out/umma/ncu_${nm}_$c.log 2>&1; echo ncu_${nm}_$c=$?
  done
done
