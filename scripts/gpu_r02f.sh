#!/bin/bash
# Round 2 session f: 3D parity, compute-sanitizer on the bulk-copy / mbarrier kernels, bench lines.
set -u
OUT=gpurun_out/r02f
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_3d.py -m gpu -q > $OUT/pytest_3d.log 2>&1; echo "pytest 3d rc=$?" | tee -a $OUT/summary.txt
tail -15 $OUT/pytest_3d.log
for T in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize_run.py > $OUT/sanitize_$T.log 2>&1
  echo "sanitize $T rc=$?" | tee -a $OUT/summary.txt
  tail -3 $OUT/sanitize_$T.log
done
HBPDC_GJ_NB=16 timeout 300 python -m pytest tests/test_gpu_br2.py -m gpu -q -k "end_of_run and gll" > $OUT/br2_nb16.log 2>&1; echo "br2 nb16 rc=$?" | tee -a $OUT/summary.txt
HBPDC_TRACE=1 timeout 300 python -m pytest tests/test_gpu_br2.py -m gpu -q -k "end_of_run and gll" > $OUT/br2_trace.log 2>&1; echo "br2 trace rc=$?" | tee -a $OUT/summary.txt
