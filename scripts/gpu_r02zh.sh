#!/bin/bash
# Round 2 session zh: end-of-round evidence for the final code -- full GPU suite, smoke, the default bench
# line (C3, as the driver runs it) + reference arm, C5 / T3 / C4 lines, the ncu launch list of a one-step C3
# run and `ncu --set full` captures of the dominant kernels, summarised on the box.
set -u
TAG=r02zh
OUT=gpurun_out/$TAG
mkdir -p $OUT /tmp/ncu_$TAG
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/summary.txt; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?" | tee -a $OUT/summary.txt
python -c "import json; d=json.load(open('$OUT/bench_c3.json')); print('C3', d['value'], d['ms_per_step'], d['roofline'], d['step_roofline']['frac'], d['solver'])" | tee -a $OUT/summary.txt
timeout 900 python bench.py --impl reference > $OUT/bench_c3_ref.json 2> $OUT/bench_c3_ref.err; echo "bench ref rc=$?" | tee -a $OUT/summary.txt
timeout 1200 python bench.py --config C5 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" | tee -a $OUT/summary.txt
python -c "import json; d=json.load(open('$OUT/bench_c5.json')); print('C5', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['solver'])" | tee -a $OUT/summary.txt
timeout 1200 python bench.py --config T3 --steps 2 --warmup 1 > $OUT/bench_t3.json 2> $OUT/bench_t3.err; echo "bench t3 rc=$?" | tee -a $OUT/summary.txt
python -c "import json; d=json.load(open('$OUT/bench_t3.json')); print('T3', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['kernels']['build'])" | tee -a $OUT/summary.txt
timeout 1500 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 rc=$?" | tee -a $OUT/summary.txt
python -c "import json; d=json.load(open('$OUT/bench_c4.json')); print('C4', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['kernels']['build'])" | tee -a $OUT/summary.txt
SHORT="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --profile-steps 0"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
    --log-file /tmp/ncu_$TAG/launches.csv $SHORT > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?" | tee -a $OUT/summary.txt
python scripts/ncu_summary.py launches /tmp/ncu_$TAG/launches.csv $OUT/launches_summary.md > /dev/null 2>&1
gzip -c /tmp/ncu_$TAG/launches.csv > $OUT/launches.csv.gz
for KS in "gemv_dmma_kernel<\(int\)6>:20" "gemv_dmma_kernel<\(int\)2>:20" "block_update_dots_tma8:60" "block_dots_tma8:60" \
          "ModeJvpFD<\(int\)1, \(int\)64>:200" "gj_kernel:2"; do
  K=${KS%%:*}; S=${KS##*:}; F=$(echo $K | tr -c 'a-zA-Z0-9_\n' '_' | cut -c1-50)
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$K" -s $S -c 1 -o /tmp/ncu_$TAG/prof_$F $SHORT > $OUT/ncu_full_$F.log 2>&1
  echo "ncu full $K rc=$?" | tee -a $OUT/summary.txt
  python scripts/ncu_summary.py full /tmp/ncu_$TAG/prof_$F.ncu-rep $OUT/ncu_full_$F.md > /dev/null 2>&1
  ncu -i /tmp/ncu_$TAG/prof_$F.ncu-rep --page raw --csv > $OUT/ncu_raw_$F.csv 2>/dev/null
done
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt; tail -3 $OUT/pytest_gpu.log
# T3 Gauss-Jordan with 320 threads (guard-free, rotated panel; build_var/libhbpdc_t320.so) vs the default 384
for V in default t320 default t320; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  HBPDC_LIB=$PWD/$L timeout 900 python bench.py --config T3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_t3_$V.json 2> $OUT/bench_t3_$V.err; echo "bench t3 $V rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_t3_$V.json'));print('T3 $V', d['value'], d['ms_per_step'], d['kernels']['build'])" | tee -a $OUT/summary.txt
done
HBPDC_LIB=$PWD/build_var/libhbpdc_t320.so timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q > $OUT/pytest_3d_t320.log 2>&1; echo "pytest 3d t320 rc=$?" | tee -a $OUT/summary.txt; tail -2 $OUT/pytest_3d_t320.log
du -sh $OUT
