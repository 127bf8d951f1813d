# s22 bench line: pageable C++ drop-in before the pinned e2e, and the K1 timings
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b22.json 2> gpurun_out/b22.log; echo bench=$?
python - <<'P'
import json
d = json.loads(open('gpurun_out/b22.json').read().strip().splitlines()[-1])
e = d['e2e']
print('value', d['ms_per_step'], 'e2e', e['ms'], 'cpp', e.get('cpp_dropin_pageable', {}).get('ms'), e.get('cpp_dropin_pageable', {}).get('ms_all'))
print(json.dumps(d.get('k1_tile_conversion'), indent=1))
P
