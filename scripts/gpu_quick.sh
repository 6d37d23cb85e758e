#!/bin/bash
# quick GPU check: build, a test subset, one short bench line
# Usage: gpurun -- bash scripts/gpu_quick.sh TAG "pytest -k expr" [bench args]
TAG=${1:-q}; K=${2:-sstep}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline "$@" > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$OUT/bench.json')); print('ms/step', d['ms_per_step']); print({k:(v['launches'],round(v['ms']),v['GBps']) for k,v in d['kernels'].items()}); print(d['solver'])"
