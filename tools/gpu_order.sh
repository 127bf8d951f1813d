# vertex-order parity + A/B of the device solve per config and order
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_order.py -x -q > gpurun_out/pytest_order.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_order.txt
for spec in "rmat22 none" "rmat22 degree" "rgg spatial" "rmat26 degree"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --order $2 --no-e2e --no-cpu-baseline > gpurun_out/ord_$1_$2.json 2> gpurun_out/ord_$1_$2.log; echo "$1 $2 rc=$?"
  python - "$1" "$2" <<'P'
import json, sys
c, o = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f'gpurun_out/ord_{c}_{o}.json').read().strip().splitlines()[-1])
    ks = sorted(d['kernels_ms'], key=lambda k: -k[2])[:6]
    print(f"{c:7s} {o:8s} value_ms {d['ms_per_step']:.4f} device_ms {d['device_resident']['ms']:.4f} order_ms {d['config']['vertex_order_ms']} |MIS| {d['config']['mis_size']} it {d['config']['iterations']} top {ks}")
except Exception as e:
    print(c, o, 'failed', e)
P
done
