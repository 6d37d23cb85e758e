#!/bin/bash
# Round 2 session t: MINB=3 (no register spills in the FD JVP) vs default MINB=4
set -u
OUT=gpurun_out/r02t
mkdir -p $OUT
for V in default m3; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  HBPDC_LIB=$L timeout 600 python scripts/op_times.py C3 20 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
done
cut -c1-400 $OUT/op_times.jsonl
