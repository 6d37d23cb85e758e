#!/bin/bash
OUT=gpurun_out/g6; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemvN_tma_kernel.*6>" -s 3 -c 1 -o $OUT/prof_g6 $SHORT > $OUT/ncu.log 2>&1
echo "ncu rc=$?"; tail -2 $OUT/ncu.log
