#!/bin/bash
# final check: build, smoke, full GPU test suite, default bench line, torchrun self-halo bench
OUT=gpurun_out/final; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['jvp']['dof_applies_per_s'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29519 \
    bench.py --gpus 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --self-halo > $OUT/torchrun.json 2> $OUT/torchrun.err
echo "torchrun rc=$?"; head -c 300 $OUT/torchrun.json
