#!/bin/bash
# Round 2 session k: GEMV row-block layout per m (C5 m = 144), parity + timings + bench lines.
set -u
OUT=gpurun_out/r02k
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchpath.py tests/test_gpu_fullsize.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest.log
timeout 600 python scripts/op_times.py C5 20 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
HBPDC_GEMV_RB2=1 timeout 600 python scripts/op_times.py C5 20 | sed 's/^{/{"variant": "rb2", /' >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
cat $OUT/op_times.jsonl | cut -c1-400
timeout 900 python bench.py --config C5 --steps 4 --warmup 2 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" | tee -a $OUT/summary.txt
timeout 400 python bench.py --steps 5 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?" | tee -a $OUT/summary.txt
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 1 > $OUT/bench_gpus2.log 2>&1; echo "bench gpus2 rc=$? (1 GPU box: expect a clean refusal)" | tee -a $OUT/summary.txt
tail -3 $OUT/bench_gpus2.log
