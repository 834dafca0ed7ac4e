python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for n in 148 0 32 74 296 444 148; do
  SIMULI_LIDAR_VARIANT=9 SIMULI_LIDAR_NLONG=$n timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nlong $n', round(d['value']/1e6,1), {k: round(v['median']*1e3,1) for k,v in d['stage_ms_distribution'].items() if isinstance(v,dict)}, 'render_tp', round(d['stages_inflight']['render']['ms_per_launch']*1e3,1))"
done
