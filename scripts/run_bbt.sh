make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/bbt
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/bench_block_tma.cu paper_2109_04804_b200/csrc/build/sstep.o paper_2109_04804_b200/csrc/build/sstep_tma.o paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/bbt && for i in 1; do timeout 300 /tmp/bbt | tee gpurun_out/bbt/out$i.txt | grep "fused\|gram\|check" | cut -c1-150; done
