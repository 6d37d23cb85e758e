#!/bin/bash
# session r02zg3: Gauss-Jordan with the pipelined update + redux pivot search + rotated panel (variant lib gjx11):
# parity of every build / precond test (K reuse off: its kk_gemm fix is still compiling) and an ncu full capture at C3
OUT=gpurun_out/r02zg3; mkdir -p $OUT /tmp/ncu_r02zg3
export HBPDC_LIB=$PWD/build_var/libhbpdc_gjx11.so
HBPDC_NS_KREUSE=0 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_errors.py tests/test_gpu_benchpath.py tests/test_gpu_fullsize.py tests/test_gpu_gl.py tests/test_gpu_br2.py -m gpu -q -k "precond or bjext or build or gj or singular or nan or benchpath or end_of_run" > $OUT/pytest_gjx11.log 2>&1; echo "pytest gjx11 rc=$?"; tail -4 $OUT/pytest_gjx11.log
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --profile-steps 0"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gj_kernel" -s 2 -c 1 -o /tmp/ncu_r02zg3/prof_gj $SHORT > $OUT/ncu_full_gj.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py full /tmp/ncu_r02zg3/prof_gj.ncu-rep $OUT/ncu_full_gj_kernel.md > /dev/null 2>&1; cat $OUT/ncu_full_gj_kernel.md
ncu -i /tmp/ncu_r02zg3/prof_gj.ncu-rep --page raw --csv > $OUT/ncu_raw_gj_kernel.csv 2>/dev/null
