#!/bin/bash
# Round 2 session o: source-level ncu captures (stall sampling per line) of the operator kernels,
# the Gauss-Jordan build and the fused s-step kernel, for the round-2 kernel work.
set -u
TAG=r02o
OUT=gpurun_out/$TAG
mkdir -p $OUT /tmp/ncu_$TAG
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
S3="python scripts/op_times.py C3 3"
S5="python scripts/op_times.py C5 3"
B3="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --profile-steps 0"
cap() {   # cap <regex> <skip> <cmd...>
  local K=$1 S=$2; shift 2
  local F=$(echo $K | tr -c 'a-zA-Z0-9_\n' '_' | cut -c1-60)
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$K" -s $S -c 1 -o /tmp/ncu_$TAG/prof_$F "$@" > $OUT/ncu_full_$F.log 2>&1
  echo "ncu full $K rc=$?" | tee -a $OUT/summary.txt
  python scripts/ncu_summary.py full /tmp/ncu_$TAG/prof_$F.ncu-rep $OUT/ncu_full_$F.md > /dev/null 2>&1
  ncu -i /tmp/ncu_$TAG/prof_$F.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/ncu_sass_$F.csv.gz
  ncu -i /tmp/ncu_$TAG/prof_$F.ncu-rep --page source --csv --print-source cuda > $OUT/ncu_src_$F.csv 2>/dev/null
}
cap 'ModeJvpFD<\(int\)1, \(int\)64>' 3 $S3
cap 'ModeKApply<\(int\)1, \(int\)64>' 1 $S3
cap 'op_kernel<\(int\)2, \(int\)2, \(int\)6, ModeJvpFD' 3 $S5
cap 'gj_kernel' 0 $S3
cap 'block_update_dots_tma8' 2 $B3
du -sh $OUT
