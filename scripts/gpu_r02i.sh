#!/bin/bash
# Round 2 session i: 3D parity after the dy fix, then the whole GPU suite.
set -u
OUT=gpurun_out/r02i
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q > $OUT/pytest_3d.log 2>&1; echo "pytest 3d rc=$?" | tee -a $OUT/summary.txt
tail -12 $OUT/pytest_3d.log
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_3d.py > $OUT/pytest_gpu.log 2>&1; echo "pytest all rc=$?" | tee -a $OUT/summary.txt
tail -8 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/summary.txt
