# full GPU parity suite + the tile Phase 1 grid A/B
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.txt; grep FAILED gpurun_out/pytest_gpu.txt | head
for spec in "grid tile auto" "rgg_spatial_ids tile auto"; do
  set -- $spec
  timeout 240 python bench.py --config $1 --candidates $2 --exclusion $3 --order none --no-e2e --no-cpu-baseline --no-k1 > gpurun_out/tc_$1_$2_$3.json 2> gpurun_out/tc_$1_$2_$3.log; echo "$1 $2 $3 rc=$?"
  python - "$1" "$2" "$3" <<'P'
import json, sys
from collections import defaultdict
c, o, x = sys.argv[1:4]
d = json.loads(open(f'gpurun_out/tc_{c}_{o}_{x}.json').read().strip().splitlines()[-1])
r1 = sorted([k for k in d['kernels_ms'] if k[1] == 1 and k[2] > 0.0068], key=lambda k: -k[2])
per = defaultdict(float)
for k, rd, ms in d['kernels_ms']: per[rd] += ms
print(c, o, x, d['device_resident']['ms'], dict((k, round(v, 4)) for k, v in sorted(per.items())), r1)
P
done
