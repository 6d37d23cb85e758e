# micro-benchmark of the S GEMV, linalg.cu variants (-D flags)
make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
C=paper_2109_04804_b200/csrc
for V in ""; do
  echo "== $V"
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a $V -I$C -c $C/linalg.cu -o /tmp/linalg_v.o && \
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude scripts/bench_gemv.cu /tmp/linalg_v.o -o /tmp/bg_v && \
  cuobjdump -res-usage /tmp/linalg_v.o | grep -A1 "gemv_dmma_kernelILi6E" | grep -o "REG:[0-9]*\|STACK:[0-9]*" ; timeout 120 /tmp/bg_v
done
