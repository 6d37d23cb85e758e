#!/bin/bash
# Round 2 session r: chunk-resident fused s-step kernel (A/B in the C3 bench kernel table), s-step parity.
set -u
OUT=gpurun_out/r02r
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sstep or s8 or s4 or batched or lock" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for F in 0 1; do
  HBPDC_FUSED_L2=$F timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_c3_l2$F.json 2> $OUT/bench_c3_l2$F.err; echo "bench l2=$F rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_c3_l2$F.json'));print($F, d['value'], d['ms_per_step'], {k:(v['ms'],v.get('GBps')) for k,v in d['kernels'].items()})"
done
