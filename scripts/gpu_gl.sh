#!/bin/bash
# GL nodes on the GPU (incl. partitions, NS) + GLL regression (parity, partition)
OUT=gpurun_out/gl; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_gl.py -q > $OUT/pytest_gl.log 2>&1; echo "gl rc=$?"; tail -25 $OUT/pytest_gl.log
timeout 1200 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py -q -x > $OUT/pytest_reg.log 2>&1; echo "reg rc=$?"; tail -3 $OUT/pytest_reg.log
