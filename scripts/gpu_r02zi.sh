#!/bin/bash
# session r02zi: m = 320 Gauss-Jordan with 320 threads as the default -- smoke, 3D / build / error-path tests, T3 line
OUT=gpurun_out/r02zi; mkdir -p $OUT
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 1200 python bench.py --config T3 --steps 2 --warmup 1 > $OUT/bench_t3.json 2> $OUT/bench_t3.err; echo "bench t3 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_t3.json')); print('T3', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['kernels']['build'])"
timeout 1500 python -m pytest tests/test_gpu_3d.py tests/test_gpu_errors.py -m gpu -q > $OUT/pytest_3d_errors.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_3d_errors.log
