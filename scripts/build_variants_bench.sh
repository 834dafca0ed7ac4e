#!/bin/bash
# compile-time variant sweep with the headline bench (in-flight rays/s) and the stage times
while IFS= read -r v; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" || { echo "build failed: $v"; continue; }
  TAG="[$v]" timeout 200 python scripts/bench_stages.py B
  timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v] headline', round(d['value']/1e6,1), 'M rays/s', round(d['ms_per_step'],4), 'ms/scan')"
done < "$1"
python -c "import paper_2510_12901_b200.build as b; b.build(force=True)"
