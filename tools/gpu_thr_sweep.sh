# device-resident solve time vs the k_tail threshold (TCMIS_TAIL_THRESHOLD)
mkdir -p gpurun_out
for c in rmat22 er grid rgg rmat26; do
  for t in 2048 8192 16384 32768 65536; do
    TCMIS_TAIL_THRESHOLD=$t timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/thr_${c}_$t.json 2>/dev/null
    echo "$c thr=$t $(python -c "import json,sys; d=json.loads(open('gpurun_out/thr_${c}_$t.json').read().strip().splitlines()[-1]); print(d['device_resident']['ms'], d['ms_per_step'])")"
  done
done
