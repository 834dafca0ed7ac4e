#!/bin/bash
# Full ncu capture of the bin_sort kernels on a synthetic case of scripts/bench_sort.py
# Usage: bash scripts/ncu_sort.sh <case> <kernel regex> [skip]
mkdir -p gpurun_out/sortprof
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s ${3:-12} -c 2 \
  -o gpurun_out/sortprof/$1 python scripts/bench_sort.py $1 > gpurun_out/sortprof/$1.log 2>&1
