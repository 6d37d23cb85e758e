make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/bbt
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a scripts/bench_block_tma.cu paper_2109_04804_b200/csrc/build/sstep.o paper_2109_04804_b200/csrc/build/sstep_tma.o paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/bbt || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:${1:-dots_tma8} -s ${2:-21} -c 1 -o gpurun_out/bbt/prof_${1:-dots_tma8} /tmp/bbt > gpurun_out/bbt/ncu_${1:-dots_tma8}.log 2>&1; echo rc=$?
tail -3 gpurun_out/bbt/ncu_${1:-dots_tma8}.log
