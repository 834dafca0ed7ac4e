python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for pdl in 1 0; do
  SIMULI_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl', round(d['value']/1e6,1), 'lat', round(d['latency_mode']['scan_ms_median']*1e3,1), {k: (round(v['value']/1e6,1), round(v['ms_per_step']*1e3,1)) for k,v in d['secondary'].items()})"
done
