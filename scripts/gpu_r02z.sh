#!/bin/bash
# Round 2 session z: Gauss-Jordan with double-buffered pivot-row tiles (cp.async) and early
# accumulator loads vs the previous kernel: BJ_ext build times (C3, C5), build parity.
set -u
OUT=gpurun_out/r02z
mkdir -p $OUT
for V in gjold default; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  for C in C3 C5 T3; do
    HBPDC_LIB=$L timeout 600 python scripts/op_times.py $C 5 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
cut -c1-300 $OUT/op_times.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_3d.py -m gpu -q -x -k "precond or bjext or build or gj" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
