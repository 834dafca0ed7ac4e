#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md): plain run first, then the tool.
# Usage (repo root, on a gpurun box): bash scripts/sanitize.sh <memcheck|racecheck|synccheck|initcheck> [--quick]
tool=$1; shift
out=gpurun_out/r02_san; mkdir -p $out
python -c "import paper_2510_12901_b200.build as b; b.build()" > $out/build_$tool.log 2>&1 || exit 1
timeout 600 python scripts/sanitize_run.py "$@" > $out/plain_$tool.log 2>&1 || { echo "plain run failed"; tail $out/plain_$tool.log; exit 1; }
extra=""
[ "$tool" = "racecheck" ] && extra="--racecheck-report all"
timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 50 \
  python scripts/sanitize_run.py "$@" > $out/$tool.log 2>&1
echo "$tool rc=$?" >> $out/$tool.log
tail -25 $out/$tool.log
