python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for pdl in 1 0 1 0; do
  SIMULI_PDL=$pdl timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl', round(d['value']/1e6,1), {k: round(v['median']*1e3,1) for k,v in d['stage_ms_distribution'].items() if isinstance(v,dict)}, 'lat', round(d['latency_mode']['scan_ms_median']*1e3,1), 'tp', {k: round(v['ms_per_launch']*1e3,1) for k,v in d['stages_inflight'].items() if isinstance(v,dict)})"
done
SIMULI_PDL=1 python scripts/sort_cmp.py; SIMULI_PDL=0 python scripts/sort_cmp.py
