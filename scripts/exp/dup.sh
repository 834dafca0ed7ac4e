python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sort or cull or full or invariance" 2>&1 | tail -2
bash scripts/sort_build_variants.sh scripts/variants/dup_items.txt
printf "0 0 6\n" > scripts/exp/h.txt
bash scripts/headline_sweep.sh scripts/exp/h.txt
