# drop-in e2e: C++ harness on pageable std::vector storage + the parity tests of the upload paths
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_parity.py -x -q -k "dropin or upload or golden_small or run_mis" > gpurun_out/pytest_e2e.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_e2e.txt
timeout 900 python bench.py --config rmat22 --no-cpu-baseline > gpurun_out/e2e_rmat22.json 2> gpurun_out/e2e_rmat22.log; echo bench=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/e2e_rmat22.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'dev', d['device_resident']['ms'])
e=d['e2e']; print('e2e pinned ms', e['ms'], e['breakdown_ms']); print('cpp', e.get('cpp_dropin_pageable'))
P
for t in 1 4 8 16; do
  TCMIS_STAGE_THREADS=$t ./e2e_probe 2>/dev/null
done
