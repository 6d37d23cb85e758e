#!/bin/bash
# session r02zg: fused s-step kernel, transient DMMA accumulator chains in phase D (TF_DCH = 1, 2, 4)
OUT=gpurun_out/r02zg; mkdir -p $OUT
C=paper_2109_04804_b200/csrc
for V in "-DTF_DCH_=1" "-DTF_DCH_=2" "-DTF_DCH_=4" "-DTF_DCH_=2 -DTF_MAXT_=16" "-DTF_DCH_=4 -DTF_MAXT_=16"; do
  echo "== $V" | tee -a $OUT/bbt_var.txt
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a $V -I$C -Iinclude --expt-relaxed-constexpr scripts/bench_block_tma.cu $C/sstep_tma.cu $C/build/sstep.o $C/build/linalg.o -o /tmp/bbv 2>&1 | grep -i error
  timeout 300 /tmp/bbv | grep "fused\|check" | cut -c1-150 | tee -a $OUT/bbt_var.txt
done
# Gauss-Jordan: pipelined trailing update (GJ_PIPE=1, default lib) vs the previous loop (build_var/libhbpdc_gjp0.so)
for V in gjp0 default gjrot1 gjrot2 gjp0 default gjrot1 gjrot2; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  for CF in C3 C5; do
    HBPDC_LIB=$PWD/$L timeout 600 python scripts/op_times.py $CF 3 | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/op_times.jsonl 2>> $OUT/op_times.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02zg/op_times.jsonl"):
    d = json.loads(l); print(d["variant"], d["config"], round(d["precond_build_ms"], 1))
PY
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_3d.py tests/test_gpu_errors.py tests/test_gpu_benchpath.py -m gpu -q -x -k "precond or bjext or build or gj or singular or nan or benchpath" > $OUT/pytest_gj.log 2>&1; echo "pytest gj rc=$?"; tail -2 $OUT/pytest_gj.log
HBPDC_LIB=$PWD/build_var/libhbpdc_gjrot2.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_errors.py tests/test_gpu_benchpath.py -m gpu -q -x -k "precond or bjext or build or gj or singular or nan or benchpath" > $OUT/pytest_gjrot2.log 2>&1; echo "pytest gjrot2 rc=$?"; tail -2 $OUT/pytest_gjrot2.log
for V in gjp0 default gjrot2; do
  if [ $V = default ]; then L=paper_2109_04804_b200/libhbpdc.so; else L=build_var/libhbpdc_$V.so; fi
  HBPDC_LIB=$PWD/$L timeout 900 python bench.py --config T3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_t3_$V.json 2> $OUT/bench_t3_$V.err; echo "bench t3 $V rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_t3_$V.json'));print('T3 $V', d['value'], d['ms_per_step'], d['kernels']['build'])"
done
# NS: K_i reused by the second build of a step (bitwise test, NS suites, C5 bench + launch list)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_br2.py tests/test_gpu_gl.py tests/test_gpu_fullsize.py -m gpu -q -x -k "ns or navier or c5 or C5" > $OUT/pytest_ns.log 2>&1; echo "pytest ns rc=$?"; tail -3 $OUT/pytest_ns.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_c5.json')); print('C5', d['value'], d['ms_per_step'], d['step_roofline'], d['solver']); print(d['kernels'])"
HBPDC_NS_KREUSE=0 timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_c5_noreuse.json 2> $OUT/bench_c5_noreuse.err; echo "c5 noreuse rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_c5_noreuse.json')); print('C5 no reuse', d['value'], d['ms_per_step'], d['solver'])"
mkdir -p /tmp/ncu_r02zg
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file /tmp/ncu_r02zg/launches_c5.csv \
  python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --profile-steps 0 > $OUT/ncu_launches_c5.log 2>&1; echo "ncu c5 rc=$?"
python scripts/ncu_summary.py launches /tmp/ncu_r02zg/launches_c5.csv $OUT/launches_c5.md > /dev/null 2>&1; head -30 $OUT/launches_c5.md
