#!/bin/bash
# render-only timing + output comparison across kernels: args = SIMULI_LIDAR_RENDER[:SIMULI_LIDAR_VARIANT] specs
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
rm -f /tmp/rv_*.npz
for k in ${@:-split}; do
  kern=${k%%:*}; var=${k#*:}; [ "$var" = "$k" ] && var=0
  SIMULI_LIDAR_RENDER=$kern SIMULI_LIDAR_VARIANT=$var python scripts/bench_render.py ${CFG:-B} /tmp/rv_$k.npz
done
python - <<'PY'
import numpy as np, glob
fs = sorted(glob.glob("/tmp/rv_*.npz")); base = np.load(fs[0])
for f in fs[1:]:
    d = np.load(f)
    print(f, {k: float(np.abs(d[k].astype(np.float64) - base[k]).max()) for k in d.files if k in base.files})
PY
