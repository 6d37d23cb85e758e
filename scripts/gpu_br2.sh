#!/bin/bash
OUT=gpurun_out/br2; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_br2.py -q > $OUT/pytest_br2.log 2>&1; echo "br2 rc=$?"; tail -30 $OUT/pytest_br2.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gl.py tests/test_gpu_partition.py -q -k "navier or ns or NS" > $OUT/pytest_ns.log 2>&1; echo "ns reg rc=$?"; tail -3 $OUT/pytest_ns.log
