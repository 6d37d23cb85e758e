#!/bin/bash
# gpurun: ncu launch list of one bench step + `ncu --set full` captures of the
# dominant kernels (Arnoldi dots/update, BJ_ext GEMV (6 RHS), FD-JVP operator).
#   gpurun --timeout 2400 -- bash scripts/gpu_profile.sh TAG
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || exit 1
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 400 $SHORT > $OUT/short_plain.log 2>&1 || { echo plain run failed; tail $OUT/short_plain.log; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 4000 --csv \
    --log-file $OUT/launches.csv $SHORT > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"dcgs2|gemvN|ModeJvpFD|ModeKApply" -s 400 -c 6 -o $OUT/prof_top $SHORT > $OUT/ncu_full.log 2>&1
echo "full rc=$?"; tail -2 $OUT/ncu_full.log
