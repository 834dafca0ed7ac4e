#!/bin/bash
# Per-kernel device times of simuli_bin_sort on synthetic lists (ncu launch list), + correctness
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
mkdir -p gpurun_out/sl
for c in ${@:-u256 u4096 o18000}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sl/$c.csv python scripts/bench_sort.py $c > /dev/null 2>&1
done
python -m pytest tests -m gpu -x -q -k "bin_sort or cull" 2>&1 | tail -2
