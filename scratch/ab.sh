# A/B: run bench summary for each config
for c in "$@"; do timeout 600 python bench.py --config $c --no-cpu-baseline $BENCH_EXTRA 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['config']['graph'], 'ms', d['ms_per_step'], 'Gedges/s', d['value'], 'frac', (d['roofline'] or {}).get('frac'), 'e2e_ms', d['e2e']['ms'], d['e2e'].get('breakdown_ms'), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
print('   ', ' '.join(f'{k}[{r}]={ms*1000:.0f}' for k,r,ms in d['kernels_ms'][:12]))
"; done
