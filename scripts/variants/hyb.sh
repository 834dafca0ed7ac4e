#!/bin/bash
python -c "import paper_2510_12901_b200.build as b; b.build()" > /dev/null || exit 1
python scripts/bench_render.py B /tmp/rv_ref.npz
for nl in 0 74 148 296 600; do
  SIMULI_LIDAR_VARIANT=9 SIMULI_LIDAR_NLONG=$nl python scripts/bench_render.py B /tmp/rv_h$nl.npz
  SIMULI_LIDAR_VARIANT=9 SIMULI_LIDAR_NLONG=$nl timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nlong $nl headline', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'latency', round(d['latency_ms_per_scan'],4))"
done
python - <<'PY'
import numpy as np, glob
a = np.load("/tmp/rv_ref.npz")
for f in sorted(glob.glob("/tmp/rv_h*.npz")):
    b = np.load(f); print(f, max(float(np.abs(a[k].astype(float) - b[k]).max()) for k in a.files))
PY
