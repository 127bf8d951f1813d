mkdir -p gpurun_out/r1
timeout 900 python -m pytest tests/test_gpu_order.py -x -q > gpurun_out/r1/pytest_order.txt 2>&1; echo pytest=$?; tail -3 gpurun_out/r1/pytest_order.txt
for c in rmat22 rmat26; do
  for v in settle nosettle; do
    envs="X=1"; [ $v = nosettle ] && envs="TCMIS_NO_R1_SETTLE=1"
    env $envs timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 5 --config $c > gpurun_out/r1/${c}_$v.json 2> gpurun_out/r1/${c}_$v.log
    python -c "
import json; d=json.loads(open('gpurun_out/r1/${c}_$v.json').read().strip().splitlines()[-1])
print('$c $v', d['ms_per_step'], d.get('device_resident',{}).get('ms'), d['config'].get('vertex_order_ms'), [(p['phase'][:12], p['round'], p['ms']) for p in d['roofline']['phases']])"
  done
done
