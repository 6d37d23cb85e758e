#!/bin/bash
# Round 2 session p: epilogue-input prefetch + register-cap variants of the operator kernels (A/B on
# C3 and C5 op timings), parity of the default build.
set -u
OUT=gpurun_out/r02p
mkdir -p $OUT
for V in base default m5 m6; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  for C in C3 C5; do
    HBPDC_LIB=$L timeout 600 python scripts/op_times.py $C 20 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
cut -c1-420 $OUT/op_times.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchpath.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
