#!/bin/bash
# GL nodes on the GPU + a GLL regression subset + a short bench (the GLL kernels must be unchanged)
OUT=gpurun_out/gl; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_gl.py -q -x > $OUT/pytest_gl.log 2>&1; echo "gl rc=$?"; tail -15 $OUT/pytest_gl.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "rhs or residual or jvp or precond" > $OUT/pytest_reg.log 2>&1; echo "reg rc=$?"; tail -2 $OUT/pytest_reg.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['jvp'])"
