mkdir -p gpurun_out/rggdeg
timeout 900 python -m pytest tests/test_gpu_order.py -x -q 2>&1 | tail -1
for o in spatial degree; do for c in rgg; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --config $c --order $o > gpurun_out/rggdeg/${c}_$o.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/rggdeg/${c}_$o.json').read().strip().splitlines()[-1])
print('$c $o', d['ms_per_step'], d.get('device_resident',{}).get('ms'), d['config'].get('vertex_order_ms'), d['kernels_ms'][:6])"
done; done
for o in none degree; do for c in er grid; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --config $c --order $o > gpurun_out/rggdeg/${c}_$o.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/rggdeg/${c}_$o.json').read().strip().splitlines()[-1])
print('$c $o', d['ms_per_step'], d.get('device_resident',{}).get('ms'), d['config'].get('vertex_order_ms'))"
done; done
