# round-2 experiment (commit 5ae5bdc; the SIMULI_SORT_RB switch was removed afterwards)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
SIMULI_SORT_RB=10 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for rb in 8 10 8 10; do SIMULI_SORT_RB=$rb python scripts/sort_cmp.py; done
for v in 0 2561204 2561608 2562004 5121204; do echo "rb10 v$v"; SIMULI_SORT_RB=10 SIMULI_SORT_VARIANT=$v python scripts/sort_cmp.py; done
printf "0 0 6\n" > scripts/exp/h.txt
bash scripts/headline_sweep.sh scripts/exp/h.txt
SIMULI_SORT_RB=10 bash scripts/headline_sweep.sh scripts/exp/h.txt
printf "0 2561608 6\n0 2561204 6\n" > scripts/exp/h2.txt
SIMULI_SORT_RB=10 bash scripts/headline_sweep.sh scripts/exp/h2.txt
