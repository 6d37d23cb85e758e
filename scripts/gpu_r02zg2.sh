#!/bin/bash
# session r02zg2: Gauss-Jordan pivot search by warp redux (GJ_REDUX) with / without the rotated panel loop, vs the pipelined default
OUT=gpurun_out/r02zg2; mkdir -p $OUT
for V in default gjx1 gjx11 default gjx1 gjx11; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  for CF in C3 C5; do
    HBPDC_LIB=$PWD/$L timeout 600 python scripts/op_times.py $CF 3 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02zg2/op_times.jsonl"):
    d = json.loads(l); print(d["variant"], d["config"], round(d["precond_build_ms"], 1))
PY
for V in gjx1 gjx11; do
HBPDC_LIB=$PWD/build_var/libhbpdc_$V.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_errors.py tests/test_gpu_benchpath.py tests/test_gpu_fullsize.py -m gpu -q -x -k "precond or bjext or build or gj or singular or nan or benchpath" > $OUT/pytest_$V.log 2>&1; echo "pytest $V rc=$?"; tail -2 $OUT/pytest_$V.log
done
for V in default gjx1 gjx11; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  HBPDC_LIB=$PWD/$L timeout 900 python bench.py --config T3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_t3_$V.json 2> $OUT/bench_t3_$V.err; echo "bench t3 $V rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_t3_$V.json'));print('T3 $V', d['value'], d['ms_per_step'], d['kernels']['build'])"
done
