# Phase 1 tile form: parity + keep/drop A/B (grid, RGG with spatial ids, R-MAT s22)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tile_cand.py tests/test_gpu_parity.py -k "tile_phase1 or corruption or tail_threshold or long_path" -x -q > gpurun_out/pytest_tilecand.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_tilecand.txt
for spec in "grid csr auto" "grid tile auto" "rgg_spatial_ids csr auto" "rgg_spatial_ids tile auto" "er tile auto" "er csr auto"; do
  set -- $spec
  timeout 240 python bench.py --config $1 --candidates $2 --exclusion $3 --order none --no-e2e --no-cpu-baseline --no-k1 > gpurun_out/tc_$1_$2_$3.json 2> gpurun_out/tc_$1_$2_$3.log; echo "$1 $2 $3 rc=$?"
  python - "$1" "$2" "$3" <<'P'
import json, sys
c, o, x = sys.argv[1:4]
try:
    d = json.loads(open(f'gpurun_out/tc_{c}_{o}_{x}.json').read().strip().splitlines()[-1])
    r1 = sorted([k for k in d['kernels_ms'] if k[1] == 1 and k[2] > 0.0068], key=lambda k: -k[2])
    from collections import defaultdict
    per = defaultdict(float)
    for k, rd, ms in d['kernels_ms']: per[rd] += ms
    print(f"{c:16s} {o:4s} {x:9s} device_ms {d['device_resident']['ms']:.4f} build {d['config']['tile_cand_build']} it {d['config']['iterations']} per_round {dict((k, round(v, 4)) for k, v in sorted(per.items()))} round1 {r1}")
except Exception as e:
    print(c, o, x, 'failed', e)
P
done
