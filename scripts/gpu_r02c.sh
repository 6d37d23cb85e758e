#!/bin/bash
# Round 2 session c: GJ panel width A/B, colour-restricted NS build, parity of both.
set -u
OUT=gpurun_out/r02c
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_errors.py tests/test_gpu_benchpath.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_partition.py tests/test_gpu_br2.py -m gpu -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest.log
for C in C3 C5 C4; do
  for NB in 32 16; do
    HBPDC_GJ_NB=$NB timeout 600 python scripts/op_times.py $C 10 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
cat $OUT/op_times.jsonl
