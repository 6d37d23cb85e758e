#!/bin/bash
# Round 2 session e: op-kernel A/B (DMMA contraction x staged faces), C5 build / JVP launch lists,
# NS BJ^H_ext + BR2 tests.
set -u
OUT=gpurun_out/r02e
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
for V in "" _dmma _nostage _dmma_nostage; do
  HBPDC_LIB=$PWD/paper_2109_04804_b200/libhbpdc$V.so timeout 300 python scripts/op_times.py C3 30 | sed "s/^{/{\"lib\": \"$V\", /" >> $OUT/op_ab.jsonl 2>> $OUT/op_ab.err
done
cat $OUT/op_ab.jsonl | cut -c1-260
timeout 900 python -m pytest tests/test_gpu_br2.py tests/test_gpu_gl.py tests/test_gpu_errors.py -m gpu -q > $OUT/pytest1.log 2>&1; echo "pytest1 rc=$?" | tee -a $OUT/summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bjext_h or c5_shape" > $OUT/pytest2.log 2>&1; echo "pytest2 rc=$?" | tee -a $OUT/summary.txt
tail -2 $OUT/pytest1.log $OUT/pytest2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_build_c5.csv python scripts/build_only.py C5 > $OUT/ncu_b5.log 2>&1; echo "ncu b5 rc=$?" | tee -a $OUT/summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_jvp_c5.csv python scripts/jvp_c5_only.py C5 > $OUT/ncu_j5.log 2>&1; echo "ncu j5 rc=$?" | tee -a $OUT/summary.txt
python scripts/parse_launches.py $OUT/launches_build_c5.csv $OUT/launches_jvp_c5.csv > $OUT/launch_summary.txt 2>&1
cat $OUT/launch_summary.txt
timeout 1500 python scripts/eoc_anchors.py > $OUT/eoc_anchors.md 2> $OUT/eoc_anchors.err; echo "anchors rc=$?" | tee -a $OUT/summary.txt
timeout 1200 python scripts/eoc_study.py --nodes gl --flux glf > $OUT/eoc_study_gl.md 2> $OUT/eoc_gl.err; echo "eoc gl rc=$?" | tee -a $OUT/summary.txt
timeout 1500 python scripts/iteration_study.py > $OUT/iteration_study.md 2> $OUT/iter.err; echo "iter rc=$?" | tee -a $OUT/summary.txt
