#!/bin/bash
# Round 2 profiling session: ncu launch list of one C3 bench step and of one C5 step, ncu --set full
# captures of the dominant kernels (C3 and C5), summaries + fp64 / DRAM numbers for bench.py.
set -u
TAG=r02h
OUT=gpurun_out/$TAG
mkdir -p $OUT /tmp/ncu_$TAG
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
S3="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --profile-steps 0"
S5="python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --profile-steps 0"
timeout 400 $S3 > $OUT/short_c3.json 2> $OUT/short_c3.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
    --log-file /tmp/ncu_$TAG/launches_c3.csv $S3 > $OUT/ncu_launches_c3.log 2>&1; echo "ncu launches c3 rc=$?" | tee -a $OUT/summary.txt
python scripts/ncu_summary.py launches /tmp/ncu_$TAG/launches_c3.csv $OUT/launches_c3.md > /dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
    --log-file /tmp/ncu_$TAG/launches_c5.csv $S5 > $OUT/ncu_launches_c5.log 2>&1; echo "ncu launches c5 rc=$?" | tee -a $OUT/summary.txt
python scripts/ncu_summary.py launches /tmp/ncu_$TAG/launches_c5.csv $OUT/launches_c5.md > /dev/null 2>&1
cap() {   # cap <regex> <skip> <cmd...>
  local K=$1 S=$2; shift 2
  local F=$(echo $K | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$K" -s $S -c 1 -o /tmp/ncu_$TAG/prof_$F "$@" > $OUT/ncu_full_$F.log 2>&1
  echo "ncu full $K rc=$?" | tee -a $OUT/summary.txt
  python scripts/ncu_summary.py full /tmp/ncu_$TAG/prof_$F.ncu-rep $OUT/ncu_full_$F.md > /dev/null 2>&1
  ncu -i /tmp/ncu_$TAG/prof_$F.ncu-rep --page raw --csv > $OUT/ncu_raw_$F.csv 2>/dev/null
}
for KS in "gemv_dmma_kernel<\(int\)6>:20" "ModeJvpFD<1, 64>:200" "ModeKApply<1, 64>:200" "ModeResid<1, 64>:10" \
          "block_update_dots_tma8:60" "block_update_tma8_kernel:60" "block_dots_tma8:60" "gj_kernel:2"; do
  cap "${KS%%:*}" "${KS##*:}" $S3
done
for KS in "ModeJvpFD<2, 36>:20" "lift_kernel<6, ModeJvpFD:20" "kk_gemm_kernel:0" "gj_kernel:2"; do
  cap "${KS%%:*}" "${KS##*:}" $S5
done
du -sh $OUT
