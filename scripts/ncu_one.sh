#!/bin/bash
# ncu --set full of one kernel launch of a short C3 bench run
# Usage: gpurun -- bash scripts/ncu_one.sh TAG KERNEL_REGEX [SKIP]
TAG=$1; K=$2; SKIP=${3:-0}
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o $OUT/prof_$K $SHORT > $OUT/ncu_$K.log 2>&1
echo "ncu rc=$?"; tail -2 $OUT/ncu_$K.log
