#!/bin/bash
# ncu --set full captures of the operator kernels (C3: FD JVP, K-apply, residual; C5: NS FD JVP),
# summaries for profiles/ and the fp64 / DRAM figures bench.py quotes.
set -u
TAG=r02l
OUT=gpurun_out/$TAG
mkdir -p $OUT /tmp/ncu_$TAG
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
S3="python scripts/op_times.py C3 3"
S5="python scripts/op_times.py C5 3"
cap() {   # cap <regex> <skip> <cmd...>
  local K=$1 S=$2; shift 2
  local F=$(echo $K | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$K" -s $S -c 1 -o /tmp/ncu_$TAG/prof_$F "$@" > $OUT/ncu_full_$F.log 2>&1
  echo "ncu full $K rc=$?" | tee -a $OUT/summary.txt
  python scripts/ncu_summary.py full /tmp/ncu_$TAG/prof_$F.ncu-rep $OUT/ncu_full_$F.md > /dev/null 2>&1
  ncu -i /tmp/ncu_$TAG/prof_$F.ncu-rep --page raw --csv > $OUT/ncu_raw_$F.csv 2>/dev/null
  ncu -i /tmp/ncu_$TAG/prof_$F.ncu-rep --page source --csv > $OUT/ncu_src_$F.csv 2>/dev/null
}
cap 'ModeJvpFD<\(int\)1, \(int\)64>' 3 $S3
cap 'ModeKApply<\(int\)1, \(int\)64>' 1 $S3
cap 'ModeResid<\(int\)1, \(int\)64>' 3 $S3
cap 'ModeJvpFD<\(int\)2, \(int\)36>' 3 $S5
cap 'gemv_dmma_kernel<\(int\)2, \(int\)4' 2 $S5
du -sh $OUT
