#!/bin/bash
# session r02zf: selective reorthogonalisation on by default (tau 1e-12) -- full GPU suite, C3 / C5 bench, NS EOC study
OUT=gpurun_out/r02zf; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_c3.json')); print('C3', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['solver'])"
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_c5.json')); print('C5', d['value'], d['ms_per_step'], d['solver'])"
timeout 1800 python scripts/eoc_ns.py > $OUT/eoc_ns.md 2> $OUT/eoc_ns.err; echo "eoc_ns rc=$?"; tail -15 $OUT/eoc_ns.md; tail -3 $OUT/eoc_ns.err
