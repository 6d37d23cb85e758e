#!/bin/bash
# Round 2 session m: 3D with the m = 320 DMMA GEMV, T3 and C4 bench lines, C5 JVP launch list.
set -u
OUT=gpurun_out/r02m
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q > $OUT/pytest_3d.log 2>&1; echo "pytest 3d rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest_3d.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_jvp_c5.csv python scripts/jvp_c5_only.py C5 > $OUT/ncu_j5.log 2>&1; echo "ncu j5 rc=$?" | tee -a $OUT/summary.txt
python scripts/parse_launches.py $OUT/launches_jvp_c5.csv > $OUT/launch_summary.txt 2>&1; cat $OUT/launch_summary.txt
timeout 1200 python bench.py --config T3 --steps 2 --warmup 1 > $OUT/bench_t3.json 2> $OUT/bench_t3.err; echo "bench t3 rc=$?" | tee -a $OUT/summary.txt
tail -2 $OUT/bench_t3.err
timeout 1500 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 rc=$?" | tee -a $OUT/summary.txt
tail -2 $OUT/bench_c4.err
