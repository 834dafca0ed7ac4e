#!/bin/bash
# compile-time variant sweep: for each SIMULI_EXTRA_NVCC value (one per line in $1), a
# forced rebuild and the config-B stage times.  Usage: build_variants.sh variants.txt [config]
cfg=${2:-B}
while IFS= read -r v; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" || { echo "build failed: $v"; continue; }
  TAG="[$v]" timeout 200 python scripts/bench_stages.py $cfg
done < "$1"
python -c "import paper_2510_12901_b200.build as b; b.build(force=True)"
