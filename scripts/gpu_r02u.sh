#!/bin/bash
# Round 2 session u: two-threads-per-node FD JVP (fdsplit.cuh): bitwise vs op_kernel, timings, parity.
set -u
OUT=gpurun_out/r02u
mkdir -p $OUT
HBPDC_FD_SPLIT=0 timeout 300 python scripts/fd_split_check.py save /tmp/fd_a.npz > $OUT/check.log 2>&1
HBPDC_FD_SPLIT=1 timeout 300 python scripts/fd_split_check.py save /tmp/fd_b.npz >> $OUT/check.log 2>&1
python scripts/fd_split_check.py cmp /tmp/fd_a.npz /tmp/fd_b.npz >> $OUT/check.log 2>&1; echo "bitwise rc=$?"; tail -8 $OUT/check.log
for V in split0 split1 f6; do
  case $V in split0) E="HBPDC_FD_SPLIT=0";; split1) E="HBPDC_FD_SPLIT=1";; f6) E="HBPDC_LIB=build_var/libhbpdc_f6.so";; esac
  env $E timeout 600 python scripts/op_times.py C3 20 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
done
cut -c1-300 $OUT/op_times.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_benchpath.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_c3.json'));print(d['value'], d['ms_per_step'], {k:(v['ms'],v.get('GBps')) for k,v in d['kernels'].items()})"
