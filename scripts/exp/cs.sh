python -c "import paper_2510_12901_b200.build as b; b.build()" > /dev/null || exit 1
timeout 120 python scripts/exp/proj_parts.py 2>/dev/null | head -2
printf "0 0 6\n0 0 6\n" > scripts/exp/h.txt
bash scripts/headline_sweep.sh scripts/exp/h.txt
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "cull or project or full or invariance or bruteforce" 2>&1 | tail -1
