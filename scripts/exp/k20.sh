python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for s in 6 4 3 6 8; do
  timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --inflight $s --no-cpu-baseline --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K20 S$s', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1))"
done
timeout 300 python bench.py --gpus 1 --steps 200 --warmup 10 --no-cpu-baseline --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K200 S6', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1))"
