#!/bin/bash
# Round 2 session v: NS BJ_ext colour build with the one-hop lifting (ModeKNS): parity + C5 timings.
set -u
OUT=gpurun_out/r02v
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_benchpath.py tests/test_gpu_gl.py -m gpu -q -x -k "navier or ns or NS or C5" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for V in 0 1; do
  HBPDC_NS_ONEHOP=$V timeout 600 python scripts/op_times.py C5 10 | sed "s/^{/{\"onehop\": $V, /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
done
cut -c1-330 $OUT/op_times.jsonl
timeout 1200 python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_c5.json'));print(d['value'], d['ms_per_step'], {k:(v['ms'],v.get('GBps')) for k,v in d['kernels'].items()})"
