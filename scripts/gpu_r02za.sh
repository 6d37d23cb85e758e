#!/bin/bash
# Round 2 session za: Gauss-Jordan variants separately (A: double-buffered pivot-row tiles only,
# B: one barrier per column only) vs the previous kernel, BJ_ext build times (C3, C5).
set -u
OUT=gpurun_out/r02za
mkdir -p $OUT
for V in gjold gjA gjB gjold; do
  for C in C3 C5; do
    HBPDC_LIB=build_var/libhbpdc_$V.so timeout 600 python scripts/op_times.py $C 3 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02za/op_times.jsonl"):
    d = json.loads(l); print(d["variant"], d["config"], round(d["precond_build_ms"], 1))
PY
