#!/bin/bash
# gpurun: time the C3 operator kernels, then one ncu --set full capture of the
# FD-JVP / K-apply / residual operator kernels.   Usage: bash scripts/prof_ops.sh TAG
TAG=${1:-ops}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || exit 1
python scripts/jvp_only.py 10 > $OUT/timing.txt 2>&1 && cat $OUT/timing.txt && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"op_kernel" -s 6 -c 4 \
   -o $OUT/prof_ops python scripts/jvp_only.py 2 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $OUT/ncu.log
