# A/B: run bench summary for each config
for c in "$@"; do timeout 600 python bench.py --config $c --no-cpu-baseline $BENCH_EXTRA 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['graph'], d['ms_per_step'], d['value'], d['per_round_ms'], d['roofline']['frac'], d['e2e']['ms'])"; done
