printf "0 0 6\n" > scripts/exp/h.txt
for v in "-DSIMULI_L_ROTATE" "" "-DSIMULI_L_ROTATE" ""; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null || exit 1
  echo "[$v]"; timeout 120 python scripts/exp/proj_parts.py 2>/dev/null | head -1
  timeout 300 bash scripts/headline_sweep.sh scripts/exp/h.txt
done
