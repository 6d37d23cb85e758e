make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude scripts/bench_block.cu paper_2109_04804_b200/csrc/build/sstep.o paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/bb && timeout 300 /tmp/bb
