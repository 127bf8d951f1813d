mkdir -p gpurun_out/gc
timeout 1200 python -m pytest tests/test_gpu_order.py tests/test_gpu_parity.py -x -q -k "order or golden or rmat26" > gpurun_out/gc/pytest.txt 2>&1; echo pytest=$?; tail -3 gpurun_out/gc/pytest.txt
for c in rmat26 rmat22; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 5 --config $c > gpurun_out/gc/$c.json 2> gpurun_out/gc/$c.log
python -c "
import json; d=json.loads(open('gpurun_out/gc/$c.json').read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d.get('device_resident',{}).get('ms'))"
done
