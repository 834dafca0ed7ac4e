#!/bin/bash
# Full ncu capture of the named kernels (one launch each) of a short bench run.
# Usage: bash scripts/ncu_full.sh <tag> <regex of kernel names> [launch-skip]
tag=$1; re=$2; skip=${3:-12}
mkdir -p gpurun_out/$tag
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$tag/build.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c 4 \
  -o gpurun_out/$tag/full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/$tag/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/$tag/ncu_full.log
