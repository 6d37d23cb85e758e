#!/bin/bash
# ncu evidence for the current code, summarised on the box (the raw .ncu-rep
# files and the launch CSV stay there: gpurun copies back at most 64 MiB).
# Usage (here): gpurun --timeout 3600 -- bash scripts/gpu_profile_round.sh TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT /tmp/ncu_$TAG
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 400 $SHORT > $OUT/short_plain.json 2> $OUT/short_plain.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
    --log-file /tmp/ncu_$TAG/launches.csv $SHORT > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?" | tee -a $OUT/summary.txt
python scripts/ncu_summary.py launches /tmp/ncu_$TAG/launches.csv $OUT/launches_summary.md > /dev/null 2>&1
for KS in "gemv_dmma_kernel<\(int\)6>:20" "gemv_dmma_kernel<\(int\)2>:20" "block_update_dots_tma8:60" "block_dots_mma_kernel:40" \
          "block_update_tma8_kernel:60" "block_scale_w8_kernel:60" "ModeJvpFD:200" "ModeKApply:200" "gj_kernel:2"; do
  K=${KS%%:*}; S=${KS##*:}; F=$(echo $K | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$K" -s $S -c 1 -o /tmp/ncu_$TAG/prof_$F $SHORT > $OUT/ncu_full_$F.log 2>&1
  echo "ncu full $K rc=$?" | tee -a $OUT/summary.txt
  python scripts/ncu_summary.py full /tmp/ncu_$TAG/prof_$F.ncu-rep $OUT/ncu_full_$F.md > /dev/null 2>&1
  ncu -i /tmp/ncu_$TAG/prof_$F.ncu-rep --page raw --csv > $OUT/ncu_raw_$F.csv 2>/dev/null
done
du -sh $OUT
