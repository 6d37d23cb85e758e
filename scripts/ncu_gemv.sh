#!/bin/bash
OUT=gpurun_out/gd; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
for NR in 6 2; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemv_dmma_kernel<\(int\)$NR>" -s 20 -c 1 -o $OUT/prof_g$NR $SHORT > $OUT/ncu$NR.log 2>&1
echo "ncu $NR rc=$?"
done
