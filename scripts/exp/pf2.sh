printf "0 0 6\n" > scripts/exp/h.txt
for v in "" "-DSIMULI_NO_SH_PREFETCH -DSIMULI_SH_LATE_PREFETCH" "-DSIMULI_NO_SH_PREFETCH" ""; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null || exit 1
  echo "[$v]"; timeout 120 python scripts/exp/proj_parts.py 2>/dev/null | head -1
  timeout 300 bash scripts/headline_sweep.sh scripts/exp/h.txt
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_project -s 3 -c 1 python scripts/exp/proj_parts.py 2>/dev/null | grep -E "dram__bytes|gpu__time" | head -3
done
