mkdir -p gpurun_out/cb
timeout 1200 python -m pytest tests/test_gpu_order.py -x -q > gpurun_out/cb/pytest_order.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/cb/pytest_order.txt
for c in rmat22 rmat26; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 5 --config $c --order degree > gpurun_out/cb/${c}_deg2.json 2> gpurun_out/cb/${c}_deg2.log
  python -c "
import json; d=json.loads(open('gpurun_out/cb/${c}_deg2.json').read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d.get('device_resident',{}).get('ms'), d['config'].get('vertex_order_ms'))"
done
