#!/bin/bash
# GL nodes on the GPU (incl. partitions) + GLL partition regression
OUT=gpurun_out/gl; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_gl.py -q > $OUT/pytest_gl.log 2>&1; echo "gl rc=$?"; tail -25 $OUT/pytest_gl.log
timeout 900 python -m pytest tests/test_gpu_partition.py -q > $OUT/pytest_part.log 2>&1; echo "part rc=$?"; tail -3 $OUT/pytest_part.log
