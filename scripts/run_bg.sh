# micro-benchmark of the S GEMV: current linalg.o vs build/linalg_old.o (if present)
make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
for o in linalg linalg_old; do
  [ -f paper_2109_04804_b200/csrc/build/$o.o ] || continue
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude scripts/bench_gemv.cu paper_2109_04804_b200/csrc/build/$o.o -o /tmp/bg_$o && echo "== $o" && /tmp/bg_$o
done
