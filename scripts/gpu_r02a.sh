#!/bin/bash
# Round 2, first GPU session: new / changed parity tests, the full GPU suite,
# C3 / C5 / C4 bench lines.  Usage: gpurun --timeout 3000 -- bash scripts/gpu_r02a.sh
set -u
OUT=gpurun_out/r02a
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import torch; f,t=torch.cuda.mem_get_info(); print('mem free', f, 'total', t)" > $OUT/mem.txt 2>&1
make -C paper_2109_04804_b200/csrc -j8 > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_errors.py tests/test_gpu_benchpath.py -m gpu -q -s > $OUT/pytest_new.log 2>&1; echo "pytest new rc=$?" | tee -a $OUT/summary.txt
tail -5 $OUT/pytest_new.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "glf or reference_mach" > $OUT/pytest_glf.log 2>&1; echo "pytest glf rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest_glf.log
timeout 300 python bench.py --steps 3 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?" | tee -a $OUT/summary.txt
timeout 600 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" | tee -a $OUT/summary.txt
timeout 900 python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 rc=$?" | tee -a $OUT/summary.txt
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_benchpath.py > $OUT/pytest_gpu.log 2>&1; echo "pytest all rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/pytest_gpu.log
