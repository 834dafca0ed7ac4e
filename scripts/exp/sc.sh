python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "scale_covariance" 2>&1 | tail -30
