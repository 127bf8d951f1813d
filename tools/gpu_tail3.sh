mkdir -p gpurun_out/tail3
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tail3/pytest_gpu.txt 2>&1; echo pytest=$?; tail -3 gpurun_out/tail3/pytest_gpu.txt
for c in rmat22 er grid rgg; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --config $c > gpurun_out/tail3/$c.json 2> gpurun_out/tail3/$c.log
  python -c "
import json; d=json.loads(open('gpurun_out/tail3/$c.json').read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d.get('device_resident',{}).get('ms'), [ (p['round'], p['ms']) for p in d['roofline']['phases'] if 'Tail' in p['phase']])"
done
bash tools/gpu_tail_prof2.sh 2>&1 | grep "^rmat22 2\|^er 2"
