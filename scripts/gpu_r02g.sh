#!/bin/bash
# Round 2 session g: single-pass NS colour build + K^2 on DMMA, GJ 160 threads, per-mode DMMA
# contraction / staging off; parity of all builds, C3/C5 timings and bench lines.
set -u
OUT=gpurun_out/r02g
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
bash scripts/gpu_r02g2.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_br2.py tests/test_gpu_gl.py tests/test_gpu_fullsize.py -m gpu -q -k "precond or bjext or c5 or ns or navier or br2 or C5" > $OUT/pytest_ns.log 2>&1; echo "pytest ns rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest_ns.log
for C in C3 C5; do timeout 600 python scripts/op_times.py $C 20 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err; done
HBPDC_NS_TWOPASS=1 HBPDC_GJ_T256=1 timeout 600 python scripts/op_times.py C5 10 | sed 's/^{/{"variant": "twopass+gj256", /' >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
cat $OUT/op_times.jsonl | cut -c1-300
timeout 300 python bench.py --steps 3 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?" | tee -a $OUT/summary.txt
timeout 900 python bench.py --config C5 --steps 4 --warmup 2 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" | tee -a $OUT/summary.txt
timeout 1500 python scripts/eoc_anchors.py > $OUT/eoc_anchors.md 2> $OUT/eoc_anchors.err; echo "anchors rc=$?" | tee -a $OUT/summary.txt
