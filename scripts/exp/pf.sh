printf "0 0 6\n" > scripts/exp/h.txt
for v in "" "-DSIMULI_NO_SH_PREFETCH" ""; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null || exit 1
  echo "[$v]"; timeout 120 python scripts/exp/proj_parts.py | head -2
  bash scripts/headline_sweep.sh scripts/exp/h.txt
done
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
