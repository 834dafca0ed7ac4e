python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 120 python scripts/cam_frame.py | tail -1
