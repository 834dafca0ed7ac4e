#!/bin/bash
# GPU iteration loop for the LiDAR render: build, render timing (10 poses of the B-batch),
# per-item timeline (profiling build), then the GPU test suite.  Usage: gpu_render_check.sh <tag>
set -u
T=gpurun_out/$1; mkdir -p $T
python -c "import paper_2510_12901_b200.build as b; b.build()" || exit 1
timeout 120 python scripts/bench_render.py B > $T/render.log 2>&1
SIMULI_EXTRA_NVCC=-DSIMULI_RENDER_PROFILE timeout 200 python scripts/render_prof.py B > $T/prof.log 2>&1
python -c "import paper_2510_12901_b200.build as b; b.build(force=True)"
timeout 300 python -m pytest tests -m gpu -x -q > $T/tests.log 2>&1
tail -2 $T/tests.log; cat $T/render.log $T/prof.log
