#!/bin/bash
# Round 2 session d: fixes (GJ NaN pivot, plain element index for non-NS kernels), staged FD JVP faces.
set -u
OUT=gpurun_out/r02d
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 600 python scripts/op_times.py C3 20 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
cat $OUT/op_times.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -5 $OUT/pytest.log
timeout 600 python scripts/op_times.py C5 10 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?" | tee -a $OUT/summary.txt
timeout 600 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" | tee -a $OUT/summary.txt
