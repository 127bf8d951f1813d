# degree-class bounds: parity (order tests) + A/B of the bench configs
mkdir -p gpurun_out/cb
timeout 1200 python -m pytest tests/test_gpu_order.py -x -q > gpurun_out/cb/pytest_order.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/cb/pytest_order.txt
run() {  # name, env, args
  name=$1; shift; envs=$1; shift
  env $envs timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 "$@" > gpurun_out/cb/$name.json 2> gpurun_out/cb/$name.log
  python - <<PY
import json
d=json.loads(open('gpurun_out/cb/$name.json').read().strip().splitlines()[-1])
print('$name', d['ms_per_step'], d.get('device_resident',{}).get('ms'), d['config'].get('vertex_order'), d['config'].get('vertex_order_ms'), d['config'].get('iterations'), d['config'].get('mis_size'))
for p in d['roofline'].get('phases',[]): print('    ', p['phase'][:40], p['round'], p['ms'])
PY
}
run rmat22_none "X=1" --config rmat22 --order none
run rmat22_deg_nocb "TCMIS_NO_CLASS_BOUNDS=1" --config rmat22 --order degree
run rmat22_deg "X=1" --config rmat22 --order degree
run rmat26_deg_nocb "TCMIS_NO_CLASS_BOUNDS=1" --config rmat26 --order degree --steps 8
run rmat26_deg "X=1" --config rmat26 --order degree --steps 8
run er_deg "X=1" --config er --order degree
run er_none "X=1" --config er --order none
