#!/bin/bash
# compile-time sort variants: order hash + bin_sort time (L2 warm) per SIMULI_EXTRA_NVCC line of $1
while IFS= read -r v; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" || { echo "build failed: $v"; continue; }
  echo "[$v]"; python scripts/sort_check.py; python scripts/sort_cmp.py
done < "$1"
python -c "import paper_2510_12901_b200.build as b; b.build(force=True)"
