python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
printf "0 0 6\n3 0 6\n0 0 6\n" > scripts/exp/h.txt
timeout 600 bash scripts/headline_sweep.sh scripts/exp/h.txt
