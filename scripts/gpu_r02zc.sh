#!/bin/bash
# Round 2 session zc: residual on the DMMA contraction (with the fifth-k-step surface terms) vs FMA
set -u
OUT=gpurun_out/r02zc
mkdir -p $OUT
for V in default rdmma default rdmma; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  HBPDC_LIB=$L timeout 600 python scripts/op_times.py C3 20 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
done
python - <<'PY'
import json
for l in open("gpurun_out/r02zc/op_times.jsonl"):
    d = json.loads(l); print(d["variant"], round(d["residual_us"], 1), round(d["jvp_fd_us"], 1), round(d["r1_us"], 1))
PY
