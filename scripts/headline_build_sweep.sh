#!/bin/bash
# compile-time variant x runtime combos: for each SIMULI_EXTRA_NVCC line of $1, the headline sweep of $2
while IFS= read -r v; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null || { echo "build failed: $v"; continue; }
  echo "== [$v]"; bash scripts/headline_sweep.sh "$2"
done < "$1"
python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null
