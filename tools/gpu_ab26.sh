mkdir -p gpurun_out/ab26
for v in base miso; do
  envs="X=1"; [ $v = miso ] && envs="TCMIS_MIS_O_MAX=200000000"
  env $envs timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 5 --config rmat26 > gpurun_out/ab26/$v.json 2> gpurun_out/ab26/$v.log
  python -c "
import json; d=json.loads(open('gpurun_out/ab26/$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d.get('device_resident',{}).get('ms'), [(p['phase'][:12], p['round'], p['ms']) for p in d['roofline']['phases']])"
done
