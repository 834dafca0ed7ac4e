#!/bin/bash
# onesweep shape sweep: order hash + bin_sort device time (L2 warm) per SIMULI_SORT_VARIANT
python -c "import paper_2510_12901_b200.build as b; b.build()" || exit 1
for v in ${@:-0}; do
  SIMULI_SORT_VARIANT=$v timeout 120 python scripts/sort_check.py
  SIMULI_SORT_VARIANT=$v timeout 120 python scripts/sort_cmp.py
done
