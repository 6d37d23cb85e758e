#!/bin/bash
# Round 2 session j: halo/compute overlap (loopback partitions bitwise), transposed K gather,
# launch_elem in every operator kernel (timing check), then the ncu profiling session.
set -u
OUT=gpurun_out/r02j
mkdir -p $OUT
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_partition.py tests/test_gpu_3d.py tests/test_gpu_br2.py -m gpu -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -6 $OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gl.py -m gpu -q -k "precond or bjext or c5 or navier" > $OUT/pytest_ns.log 2>&1; echo "pytest ns rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest_ns.log
for C in C3 C5; do timeout 600 python scripts/op_times.py $C 20 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err; done
cat $OUT/op_times.jsonl | cut -c1-330
bash scripts/gpu_r02h.sh
