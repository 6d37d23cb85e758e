#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, the ncu launch list
# of a short bench run, and `ncu --set full` captures of the dominant kernels.
# Usage (here): gpurun --timeout 3000 -- bash scripts/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" | tee -a $OUT/summary.txt
cat $OUT/bench.json
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 400 $SHORT > $OUT/short_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file $OUT/launches.csv $SHORT > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?" | tee -a $OUT/summary.txt
for K in gemvN_tma block_dots_mma block_update_mma op_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 30 -c 1 \
      -o $OUT/prof_$K $SHORT > $OUT/ncu_full_$K.log 2>&1; echo "ncu full $K rc=$?" | tee -a $OUT/summary.txt
done
