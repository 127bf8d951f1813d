# native partitioned solve: GPU tests of the multi-GPU path + one-rank bench legs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q -s > gpurun_out/pytest_part.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_part.txt; grep "host profile" gpurun_out/pytest_part.txt | head -3
for c in rmat22; do
  timeout 600 python bench.py --partitioned --config $c --no-cpu-baseline --steps 5 > gpurun_out/part1_$c.json 2> gpurun_out/part1_$c.log; echo $c=$?
  python -c "
import json; d=json.loads(open('gpurun_out/part1_$c.json').read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d['config']['iterations'], d['config']['mis_size'], d['single_gpu_same_graph'], d['host_profile'], (d['e2e'] or {}).get('ms'))"
done
timeout 600 python tools/part_local_ab.py 22 5 > gpurun_out/part_local_ab.txt 2>&1; echo ab=$?
cat gpurun_out/part_local_ab.txt | tail -8
