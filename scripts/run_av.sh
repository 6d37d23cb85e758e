# micro-benchmark of the library's Arnoldi kernels (scripts/bench_arnoldi.cu)
make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude scripts/bench_arnoldi.cu paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/ba && timeout 300 /tmp/ba
