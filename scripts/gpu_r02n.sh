#!/bin/bash
# Round 2 session n: GL face traces for the FD JVP (parity + timing A/B).
set -u
OUT=gpurun_out/r02n
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gl.py tests/test_gpu_parity.py -m gpu -q -k "gl or GL or glf" > $OUT/pytest_gl.log 2>&1; echo "pytest gl rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest_gl.log
for T in 1 0; do HBPDC_GL_TRACES=$T timeout 600 python scripts/op_times.py C3 20 gl >> $OUT/op_times.jsonl 2>> $OUT/op_times.err; done
cat $OUT/op_times.jsonl | cut -c1-300
timeout 600 python bench.py --nodes gl --flux glf --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/bench_c3_gl.json 2> $OUT/bench_c3_gl.err; echo "bench gl rc=$?" | tee -a $OUT/summary.txt
