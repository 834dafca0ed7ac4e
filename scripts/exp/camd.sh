for v in "-DSIMULI_CAM_DENSE=1" "-DSIMULI_CAM_DENSE=2" "-DSIMULI_CAM_DENSE=3" "-DSIMULI_CAM_DENSE=4"; do
  SIMULI_EXTRA_NVCC="$v" python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null || exit 1
  echo "[$v]"; timeout 120 python scripts/cam_frame.py | tail -1; SIMULI_PER_RAY_SH=1 timeout 120 python scripts/bench_camera_render.py
done
python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null
