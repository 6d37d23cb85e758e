#!/bin/bash
# Round 2 session w: NS lift kernel without the BR2 face output (BR1 instantiations) and
# occupancy variants (HBPDC_LIFT_MINB 5 / 6 / 8) on the C5 operators; NS parity.
set -u
OUT=gpurun_out/r02w
mkdir -p $OUT
for V in default l5 l6 l8; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  HBPDC_LIB=$L timeout 600 python scripts/op_times.py C5 10 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
done
cut -c1-330 $OUT/op_times.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_br2.py tests/test_gpu_partition.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
