#!/bin/bash
# A/B timing of one source file: bench_stages.py with the working tree (A) and with
# scripts/_ab_old/<file> swapped in (B).  Usage: bash scripts/ab_file.sh <csrc file> [config]
f=$1; cfg=${2:-B}
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
TAG=new python scripts/bench_stages.py $cfg
cp paper_2510_12901_b200/csrc/$f /tmp/ab_new_$f
cp scripts/_ab_old/$f paper_2510_12901_b200/csrc/$f
python -c "from paper_2510_12901_b200 import build as B; B.build(force=True)" > /dev/null
TAG=old python scripts/bench_stages.py $cfg
cp /tmp/ab_new_$f paper_2510_12901_b200/csrc/$f
python -c "from paper_2510_12901_b200 import build as B; B.build(force=True)" > /dev/null
