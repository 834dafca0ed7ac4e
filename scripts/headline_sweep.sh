#!/bin/bash
# In-flight headline (bench.py, 300 scans) per combination "lidar_variant sort_variant inflight" (lines of $1)
python -c "import paper_2510_12901_b200.build as b; b.build()" > /dev/null || exit 1
while read -r lv sv s; do
  [ -z "$lv" ] && continue
  SIMULI_LIDAR_VARIANT=$lv SIMULI_SORT_VARIANT=$sv timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline \
    --no-secondary --inflight $s | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lv $sv $s', round(d['value']/1e6,1), round(d['ms_per_step'],4), {k: round(v['median']*1e3,1) for k,v in d['stage_ms_distribution'].items() if isinstance(v,dict)})"
done < "$1"
