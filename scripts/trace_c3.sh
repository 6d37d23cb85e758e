make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/trace
HBPDC_PRED_TAYLOR=1 HBPDC_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/trace/bench_t.json 2> gpurun_out/trace/trace_t.txt
grep -A9 "predictor stage" gpurun_out/trace/trace_t.txt | head -40
python -c "import json; d=json.load(open('gpurun_out/trace/bench_t.json')); print(d['ms_per_step'], d['solver'])"
