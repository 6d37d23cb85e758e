#!/bin/bash
# Round 2 session zb: Gauss-Jordan with the block size as a compile-time constant (guard-free for
# m = 256) vs the previous kernel; build parity (2D, 3D, full size).
set -u
OUT=gpurun_out/r02zb
mkdir -p $OUT
for V in gjold default gjold default; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  for C in C3 C5; do
    HBPDC_LIB=$L timeout 600 python scripts/op_times.py $C 3 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02zb/op_times.jsonl"):
    d = json.loads(l); print(d["variant"], d["config"], round(d["precond_build_ms"], 1))
PY
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_3d.py tests/test_gpu_errors.py tests/test_gpu_benchpath.py -m gpu -q -x -k "precond or bjext or build or gj or singular or nan or benchpath" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
timeout 900 python bench.py --config T3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_t3.json 2> $OUT/bench_t3.err; echo "bench t3 rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_t3.json'));print(d['value'], d['ms_per_step'], {k:(v['ms'],v.get('GBps')) for k,v in d['kernels'].items()})"
