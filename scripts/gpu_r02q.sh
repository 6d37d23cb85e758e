#!/bin/bash
# Round 2 session q: surface terms as a fifth DMMA k-step + per-field load pointers (A/B vs base),
# operator parity.
set -u
OUT=gpurun_out/r02q
mkdir -p $OUT
for V in base default; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  for C in C3 C5; do
    HBPDC_LIB=$L timeout 600 python scripts/op_times.py $C 20 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
  HBPDC_LIB=$L timeout 600 python scripts/op_times.py C3 20 gl | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
done
cut -c1-420 $OUT/op_times.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gl.py tests/test_gpu_benchpath.py tests/test_gpu_fullsize.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
