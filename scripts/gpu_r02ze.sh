#!/bin/bash
# session r02ze: selective reorthogonalisation trace + A/B on C3, Navier-Stokes EOC study (E8)
OUT=gpurun_out/r02ze; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "selective or sstep or batched or lift_cache" -q > $OUT/pytest_sel.log 2>&1; echo "pytest sel rc=$?"; tail -2 $OUT/pytest_sel.log
HBPDC_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 0 \
  2> $OUT/trace_c3.err > $OUT/trace_c3.json; echo "trace rc=$?"; grep "s-step blocks" $OUT/trace_c3.err | tail -1
for tau in 0 1e-13 1e-12 1e-10; do
  HBPDC_SEL_REORTH=$tau timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --profile-steps 0 \
    > $OUT/ab_$tau.json 2> $OUT/ab_$tau.err; echo "tau=$tau rc=$?"
  python -c "import json; d=json.load(open('$OUT/ab_$tau.json')); print('$tau', d['value'], d['ms_per_step'])"
done
HBPDC_SEL_REORTH=1e-12 HBPDC_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 0 \
  2> $OUT/trace_c3_sel.err > $OUT/trace_c3_sel.json; grep "s-step blocks" $OUT/trace_c3_sel.err | tail -1
grep -c "newton sys" $OUT/trace_c3.err $OUT/trace_c3_sel.err
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --profile-steps 0 > $OUT/c5.json 2> $OUT/c5.err; echo "c5 rc=$?"
python -c "import json; d=json.load(open('$OUT/c5.json')); print('C5', d['value'], d['ms_per_step'])"
timeout 1500 python scripts/eoc_ns.py > $OUT/eoc_ns.md 2> $OUT/eoc_ns.err; echo "eoc_ns rc=$?"; tail -15 $OUT/eoc_ns.md; tail -3 $OUT/eoc_ns.err
