python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
printf "0 0 6\n3 0 6\n0 0 6\n3 0 6\n0 0 8\n" > scripts/exp/h4.txt
bash scripts/headline_sweep.sh scripts/exp/h4.txt
