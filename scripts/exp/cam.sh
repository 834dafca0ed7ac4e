python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "camera or compose or smoke" 2>&1 | tail -2
timeout 120 python scripts/cam_frame.py
SIMULI_PER_RAY_SH=1 timeout 120 python scripts/bench_camera_render.py
