#!/bin/bash
set -u
OUT=gpurun_out/r02g
mkdir -p $OUT
timeout 600 python scripts/debug_3d.py > $OUT/debug_3d.log 2>&1; echo "debug3d rc=$?"
head -50 $OUT/debug_3d.log
for NB in 32 16; do HBPDC_GJ_NB=$NB timeout 300 python scripts/debug_br2.py >> $OUT/debug_br2.log 2>&1; done
cat $OUT/debug_br2.log
