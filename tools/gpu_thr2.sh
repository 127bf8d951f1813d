mkdir -p gpurun_out/thr2
for c in rmat22 er rmat26 grid; do
for t in 65536 16384 4096; do
  TCMIS_TAIL_THRESHOLD=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --config $c > gpurun_out/thr2/${c}_$t.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/thr2/${c}_$t.json').read().strip().splitlines()[-1])
print('$c $t', d['ms_per_step'], d.get('device_resident',{}).get('ms'))"
done; done
