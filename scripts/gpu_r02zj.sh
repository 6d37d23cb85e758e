#!/bin/bash
# session r02zj: ncu --set full captures of the dominant kernel (BJ_ext DMMA GEMV, 6 and 2 right-hand sides) at the final code
OUT=gpurun_out/r02zj; mkdir -p $OUT /tmp/ncu_r02zj
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --profile-steps 0"
for KS in "gemv_dmma_kernel<\(int\)6,:20:gemv6" "gemv_dmma_kernel<\(int\)2,:20:gemv2"; do
  K=${KS%%:*}; R=${KS#*:}; S=${R%%:*}; F=${R##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$K" -s $S -c 1 -o /tmp/ncu_r02zj/prof_$F $SHORT > $OUT/ncu_full_$F.log 2>&1
  echo "ncu full $K rc=$?"
  python scripts/ncu_summary.py full /tmp/ncu_r02zj/prof_$F.ncu-rep $OUT/ncu_full_$F.md > /dev/null 2>&1; cat $OUT/ncu_full_$F.md
  ncu -i /tmp/ncu_r02zj/prof_$F.ncu-rep --page raw --csv > $OUT/ncu_raw_$F.csv 2>/dev/null
done
