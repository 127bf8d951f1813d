mkdir -p gpurun_out/verify
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/verify/pytest_gpu.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/verify/pytest_gpu.txt
for c in er rmat22; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --config $c > gpurun_out/verify/$c.json 2> gpurun_out/verify/$c.log
  python -c "
import json; d=json.loads(open('gpurun_out/verify/$c.json').read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d.get('device_resident',{}).get('ms'), [k for k in d['kernels_ms'] if k[0] in ('k_tail','k_prio_settle','k_init_ctrl')])"
done
