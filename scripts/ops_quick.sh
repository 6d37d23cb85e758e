#!/bin/bash
# build, operator parity tests, C3 operator timings.  Usage: gpurun -- bash scripts/ops_quick.sh TAG [pytest -k]
TAG=${1:-ops}; K=${2:-"rhs or residual or jvp or precond"}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
python scripts/jvp_only.py 20 2>&1 | tail -8 | tee $OUT/timing.txt
