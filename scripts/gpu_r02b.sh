#!/bin/bash
# Round 2 session b: DMMA-contraction parity, error-path tests, operator micro-timings, GJ occupancy A/B,
# launch list of one C3 / C5 BJ_ext build.
set -u
OUT=gpurun_out/r02b
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_errors.py tests/test_gpu_benchpath.py tests/test_gpu_fullsize.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest.log
for C in C3 C5 C4; do
  for O in 1 2; do
    HBPDC_GJ_OCC=$O timeout 600 python scripts/op_times.py $C 20 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
cat $OUT/op_times.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_build_c3.csv python scripts/build_only.py C3 > $OUT/ncu_build_c3.log 2>&1; echo "ncu c3 rc=$?" | tee -a $OUT/summary.txt
