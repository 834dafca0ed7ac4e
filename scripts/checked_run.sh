#!/bin/bash
# Substitute for compute-sanitizer (closed on the GPU pool): a checked build (device-side
# bounds / invariant assertions, SIMULI_CHECKED) running the sanitizer workload and the GPU
# test suite, then the normal build again.  Usage (repo root, GPU box): bash scripts/checked_run.sh
out=gpurun_out/r02_checked; mkdir -p $out
SIMULI_EXTRA_NVCC=-DSIMULI_CHECKED python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > $out/build.log 2>&1 || exit 1
strings paper_2510_12901_b200/libsimuli.so | grep -c "SIMULI_CHECK failed" > $out/check_strings.txt
timeout 900 python scripts/sanitize_run.py > $out/sanitize_run.log 2>&1; echo "sanitize_run rc=$?" >> $out/sanitize_run.log
SIMULI_EXTRA_NVCC=-DSIMULI_CHECKED timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
SIMULI_EXTRA_NVCC=-DSIMULI_CHECKED timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-secondary > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
grep -h "SIMULI_CHECK failed" $out/*.log $out/bench.err | head
tail -2 $out/sanitize_run.log $out/pytest_gpu.log; tail -1 $out/bench.err
python -c "import paper_2510_12901_b200.build as b; b.build(force=True)" > /dev/null 2>&1
