#!/bin/bash
# gpurun: build, GPU tests (optionally a -k filter), optional bench.
set -u
TAG=${1:-t}; K=${2:-}; BENCH=${3:-0}
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -30 $OUT/pytest_gpu.log
if [ "$BENCH" = "1" ]; then
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -5 $OUT/bench.err
fi
