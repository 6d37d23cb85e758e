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
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
    --log-file $OUT/launches.csv $SHORT > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?" | tee -a $OUT/summary.txt
# representative launches: the 6-RHS GEMV of a corrector sweep, the fused CGS pass and the
# block dots at a grown basis, the FD JVP, the Gauss-Jordan build
for KS in "gemv_dmma_kernel<\(int\)6>:20" "gemv_dmma_kernel<\(int\)2>:20" "block_update_dots_tma8:60" "block_dots_mma_kernel:40" \
          "block_update_tma8_kernel:60" "block_scale_w8_kernel:60" "ModeJvpFD:200" "ModeKApply:200" "gj_kernel:2"; do
  K=${KS%%:*}; S=${KS##*:}; F=$(echo $K | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$K" -s $S -c 1 -o $OUT/prof_$F $SHORT > $OUT/ncu_full_$F.log 2>&1
  echo "ncu full $K rc=$?" | tee -a $OUT/summary.txt
done
# multi-GPU plumbing under torchrun (1 process, NCCL self-halo through the transport)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --self-halo > $OUT/torchrun_selfhalo.json 2> $OUT/torchrun_selfhalo.err
echo "torchrun self-halo rc=$?" | tee -a $OUT/summary.txt
