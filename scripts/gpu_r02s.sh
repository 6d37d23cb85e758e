#!/bin/bash
# Round 2 session s: resident fused s-step kernel with 64-element chunks (47-tile ring) vs the
# L2 re-stream kernel vs 128-element chunks (24-tile ring).
set -u
OUT=gpurun_out/r02s
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sstep or s8 or s4 or batched or lock" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
run() {  # run TAG env...
  local T=$1; shift
  env "$@" timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_c3_$T.json 2> $OUT/bench_c3_$T.err; echo "bench $T rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_c3_$T.json'));print('$T', d['value'], d['ms_per_step'], {k:(v['ms'],v.get('GBps')) for k,v in d['kernels'].items()})"
}
run res64 HBPDC_FUSED_L2=0
run l2 HBPDC_FUSED_L2=1
run res128 HBPDC_LIB=build_var/libhbpdc_tr128.so
