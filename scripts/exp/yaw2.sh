python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 120 python scripts/exp/proj_parts.py 2>/dev/null | head -1
printf "0 0 6\n0 0 6\n" > scripts/exp/h.txt
timeout 300 bash scripts/headline_sweep.sh scripts/exp/h.txt
