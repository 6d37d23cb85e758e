#!/bin/bash
# Round 2 session x: full GPU suite after the round-2 kernel changes (one-hop NS build incl.
# partitions, lift occupancy by jet width), C3 / C5 operator timings, C5 bench line.
set -u
OUT=gpurun_out/r02x
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
for C in C3 C5; do timeout 600 python scripts/op_times.py $C 10 >> $OUT/op_times.jsonl 2>> $OUT/op_times.err; done
cut -c1-330 $OUT/op_times.jsonl
timeout 1200 python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?"
python -c "import json;d=json.load(open('$OUT/bench_c5.json'));print(d['value'], d['ms_per_step'], {k:(v['ms'],v.get('GBps')) for k,v in d['kernels'].items()})"
