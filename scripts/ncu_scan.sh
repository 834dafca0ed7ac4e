#!/bin/bash
# ncu --set full of every kernel of one steady-state config-B scan (13 launches) -> traffic
tag=${1:-scan}
mkdir -p gpurun_out/$tag
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$tag/build.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_" -s 60 -c 12 \
  -o gpurun_out/$tag/full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/$tag/ncu_full.log 2>&1
echo "ncu rc=$?"
